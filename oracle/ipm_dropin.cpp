// oracle/ipm_dropin.cpp — end-to-end drop-in check (test infrastructure).
//
// Runs the UNMODIFIED reference interior-point driver (ipm::solve_nlp,
// ipm/solver.hpp:469) on the multi-period OPF with the B200 path plugged in
// through the reference's own seams:
//   --nlp cuda : gridnlp_b200::CudaOpfNlp (NlpProblem over the C-ABI)
//   --nlp ref  : the reference's PatternNlp (CPU tape callbacks)
// In both cases the condensed KKT is the shim CondensedKkt
// (include/gridnlp_b200/shim, found first on the include path), i.e. the B200
// set_jacobian/assemble feeding the reference LDL^T.  Prints one JSON line.
//
// Input: a binary network file written by tests/test_dropin.py (SoA arrays
// in the order of gn_network, then the T x n_load demand table).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gridnlp/ipm/condensed.hpp"  // resolves to the shim
#include "gridnlp/ipm/pattern_nlp.hpp"
#include "gridnlp/ipm/solver.hpp"
#include "gridnlp/power/network.hpp"
#include "gridnlp/power/opf.hpp"
#include "gridnlp_b200/cuda_opf_nlp.hpp"

#ifndef GRIDNLP_B200_CONDENSED_SHIM
#error "the shim condensed.hpp must shadow the reference header"
#endif

using namespace gridnlp;

namespace {

template <class T>
std::vector<T> read(std::ifstream& f, size_t n) {
  std::vector<T> v(n);
  if (n) f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(T)));
  if (!f) throw std::runtime_error("truncated network file");
  return v;
}

power::MultiPeriodCase load(const char* path) {
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

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: ipm_dropin <network.bin> cuda|ref [tol] [repeat]\n");
    return 2;
  }
  try {
    const power::MultiPeriodCase mpc = load(argv[1]);
    const std::string which = argv[2];
    ipm::SolverConfig cfg;
    cfg.tol = argc > 3 ? std::atof(argv[3]) : 1e-4;
    ipm::SolveResult r;
    // seconds = solve_nlp only (the problem object is built first, as gnr_solve does);
    // with `repeat` > 1 the solve runs again on the same problem object and
    // warm_seconds times the last one (one-time CUDA module loading etc. excluded)
    const int repeat = argc > 4 ? std::max(1, std::atoi(argv[4])) : 1;
    double secs = 0.0, warm = 0.0;
    auto timed = [&](auto& nlp) {
      for (int k = 0; k < repeat; ++k) {
        const auto t0 = std::chrono::steady_clock::now();
        r = ipm::solve_nlp(nlp, cfg);
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (k == 0) secs = s;
        warm = s;
      }
    };
    if (which == "cuda") {
      gridnlp_b200::CudaOpfNlp nlp(mpc);
      timed(nlp);
    } else {
      power::BuiltOpf built = power::build_multiperiod_opf(mpc);
      ipm::PatternNlp nlp(built.model);
      timed(nlp);
    }
    std::printf("{\"nlp\": \"%s\", \"iterations\": %d, \"objective\": %.17g, \"status\": \"%s\", "
                "\"restorations\": %d, \"seconds\": %.6f, \"warm_seconds\": %.6f, "
                "\"kkt_generic\": %ld, \"kkt_specialised\": %ld}\n",
                which.c_str(), r.iterations, r.objective, ipm::to_string(r.status),
                r.restorations, secs, warm, ipm::b200_kkt_counts[0], ipm::b200_kkt_counts[1]);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
