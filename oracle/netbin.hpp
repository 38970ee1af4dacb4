// oracle/netbin.hpp -- the binary network file of oracle.bindings.write_network_bin read
// into the reference's power::MultiPeriodCase (test / bench infrastructure).
#pragma once
#include <cstdint>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gridnlp/power/network.hpp"

namespace netbin {
using namespace gridnlp;
template <class T>
inline std::vector<T> read(std::ifstream& f, size_t n) {
  std::vector<T> v(n);
  if (n) f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(T)));
  if (!f) throw std::runtime_error("truncated network file");
  return v;
}

inline power::MultiPeriodCase load(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(std::string("cannot open ") + path);
  const auto hdr = read<int32_t>(f, 6);  // N L G D ref T
  const int32_t N = hdr[0], L = hdr[1], G = hdr[2], D = hdr[3], T = hdr[5];
  const double base = read<double>(f, 1)[0];
  power::NetworkData net;
  net.base_mva = base;
  net.reference_bus = hdr[4];
  auto vmin = read<double>(f, N), vmax = read<double>(f, N);
  net.vm_start = read<double>(f, N);
  net.va_start = read<double>(f, N);
  for (int32_t i = 0; i < N; ++i) {
    power::Bus b;
    b.id = i + 1;
    b.v_min = vmin[i];
    b.v_max = vmax[i];
    b.reference = (i == hdr[4]);
    net.buses.push_back(b);
  }
  auto lf = read<int32_t>(f, L), lt = read<int32_t>(f, L);
  auto lg = read<double>(f, L), lb = read<double>(f, L), ls = read<double>(f, L),
       la = read<double>(f, L), lA = read<double>(f, L);
  for (int32_t l = 0; l < L; ++l)
    net.lines.push_back(power::Line{lf[l], lt[l], lg[l], lb[l], ls[l], la[l], lA[l]});
  auto gb = read<int32_t>(f, G);
  std::vector<std::vector<double>> gv;
  for (int k = 0; k < 11; ++k) gv.push_back(read<double>(f, G));
  for (int32_t g = 0; g < G; ++g) {
    power::Generator x;
    x.bus = gb[g];
    x.p_min = gv[0][g];
    x.p_max = gv[1][g];
    x.q_min = gv[2][g];
    x.q_max = gv[3][g];
    x.ramp = gv[4][g];
    x.c2 = gv[5][g];
    x.c1 = gv[6][g];
    x.c0 = gv[7][g];
    x.p_start = gv[8][g];
    x.q_start = gv[9][g];
    (void)gv[10];
    net.generators.push_back(x);
  }
  auto db = read<int32_t>(f, D);
  auto dp = read<double>(f, D), dq = read<double>(f, D);
  for (int32_t j = 0; j < D; ++j) net.loads.push_back(power::Load{db[j], dp[j], dq[j]});
  power::MultiPeriodCase mpc;
  mpc.network = std::move(net);
  mpc.profile.periods = T;
  mpc.profile.n_loads = D;
  mpc.profile.scale = read<double>(f, static_cast<size_t>(T) * D);
  return mpc;
}


}  // namespace netbin
