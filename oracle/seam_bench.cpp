// oracle/seam_bench.cpp -- time the drop-in seams themselves (bench infrastructure).
//
// One IPM iteration's hot-path unit through the reference's OWN interfaces, exactly as
// ipm::IpmSolver drives them (solver.hpp:139-141, 157-158, 200-228): the LiftedProblem
// (the shim: device gathers over CudaOpfNlp; with GRIDNLP_B200_HOST_LIFTED=1 the
// reference's own class, host gathers) over the NlpProblem, then the CondensedKkt the
// solver constructs from the lifted COO arrays --
//     lifted.eval_f / eval_grad / eval_g / eval_jac / eval_hess(x, -y, 1)
//     kkt.set_jacobian(J_l); kkt.assemble(H_l, Sigma_x, Sigma_s, dw, dc)
// with std::vector (pageable host) spans, as the reference passes them.  The problem is
//   cuda : gridnlp_b200::CudaOpfNlp + the shim CondensedKkt (recognised as the OPF problem:
//          OPF-specialised assembly on the B200)
//   ref  : the reference's PatternNlp callbacks + the same shim CondensedKkt.
// The shim's LDL^T analysis is lazy (first factorize), so none runs here.  Prints one JSON
// line: ms per unit (median), its split, nnz per unit.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "gridnlp/ipm/condensed.hpp"  // resolves to the shim
#include "gridnlp/ipm/lifted.hpp"
#include "gridnlp/ipm/pattern_nlp.hpp"
#include "gridnlp/power/opf.hpp"
#include "gridnlp_b200/cuda_opf_nlp.hpp"
#include "netbin.hpp"

#ifndef GRIDNLP_B200_CONDENSED_SHIM
#error "the shim condensed.hpp must shadow the reference header"
#endif
#ifndef GRIDNLP_B200_LIFTED_SHIM
#error "the shim lifted.hpp must shadow the reference header"
#endif

using namespace gridnlp;
using clk = std::chrono::steady_clock;

static double secs(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

template <class Nlp>
static int run(Nlp& nlp, const char* which, int units) {
  const auto t0 = clk::now();
  ipm::LiftedProblem lifted(nlp, 1e-4);
  ipm::CondensedKkt kkt(lifted.n(), lifted.m(), lifted.jac_rows(), lifted.jac_cols(),
                        lifted.hess_rows(), lifted.hess_cols());
  const double setup = secs(t0, clk::now());
  const size_t n = static_cast<size_t>(lifted.n()), m = static_cast<size_t>(lifted.m());
  // an interior point of the lifted boxes, row weights, bound-condensation diagonals
  std::mt19937_64 rng(1234);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<double> x(n), w(m), sx(n), ss(m);
  const auto xl = lifted.x_lower(), xu = lifted.x_upper(), xs = lifted.x_start();
  for (size_t i = 0; i < n; ++i) {
    const bool box = std::isfinite(xl[i]) && std::isfinite(xu[i]);
    x[i] = box ? xl[i] + (0.15 + 0.7 * u(rng)) * (xu[i] - xl[i]) : xs[i] + 0.2 * (u(rng) - 0.5);
    sx[i] = std::pow(10.0, 4.0 * u(rng) - 2.0);
  }
  for (size_t i = 0; i < m; ++i) {
    w[i] = 2.0 * u(rng) - 1.0;
    ss[i] = std::pow(10.0, 4.0 * u(rng) - 2.0);
  }
  double f = 0.0;
  std::vector<double> grad(n), g(m), jl(static_cast<size_t>(lifted.jac_nnz())),
      hl(static_cast<size_t>(lifted.hess_nnz()));
  const double dw = 1e-4, dc = 1e-8 * std::pow(0.1, 0.25);  // the bench's retry variant
  std::vector<double> tu, tcb, tkkt;
  for (int k = 0; k < units + 1; ++k) {  // unit 0 is a warm-up
    const auto a = clk::now();
    bool ok = lifted.eval_f(x, f) && lifted.eval_grad(x, grad) && lifted.eval_g(x, g) &&
              lifted.eval_jac(x, jl) && lifted.eval_hess(x, w, 1.0, hl);
    const auto b = clk::now();
    kkt.set_jacobian(jl);
    kkt.assemble(hl, sx, ss, dw, dc);
    volatile double sink = kkt.jacobian_values()[0];  // A has landed on the host, too
    (void)sink;
    const auto c = clk::now();
    if (!ok) {
      std::fprintf(stderr, "evaluation failed\n");
      return 1;
    }
    if (k == 0) continue;
    tu.push_back(secs(a, c));
    tcb.push_back(secs(a, b));
    tkkt.push_back(secs(b, c));
  }
  auto med = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  const long long nj = static_cast<long long>(nlp.jac_rows().size()),
                  nh = static_cast<long long>(nlp.hess_rows().size()),
                  mn = static_cast<long long>(kkt.values().size());
  std::printf("{\"nlp\": \"%s\", \"units\": %d, \"ms_per_unit\": %.6f, \"callbacks_ms\": %.6f, "
              "\"kkt_ms\": %.6f, \"setup_s\": %.3f, \"nnz_per_unit\": %lld, \"J\": %lld, "
              "\"H\": %lld, \"M\": %lld, \"kkt_specialised\": %d, \"lifted_device\": %d}\n",
              which, units, 1e3 * med(tu), 1e3 * med(tcb), 1e3 * med(tkkt), setup,
              nj + nh + mn, nj, nh, mn, kkt.b200_specialised() ? 1 : 0,
              lifted.b200_device() ? 1 : 0);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: seam_bench <network.bin> cuda|ref [units]\n");
    return 2;
  }
  try {
    const power::MultiPeriodCase mpc = netbin::load(argv[1]);
    const std::string which = argv[2];
    const int units = argc > 3 ? std::max(1, std::atoi(argv[3])) : 3;
    if (which == "cuda") {
      gridnlp_b200::CudaOpfNlp nlp(mpc);
      return run(nlp, "cuda", units);
    }
    power::BuiltOpf built = power::build_multiperiod_opf(mpc);
    ipm::PatternNlp nlp(built.model);
    built.model.set_threads(static_cast<int>(std::max(1u, std::thread::hardware_concurrency())));
    return run(nlp, "ref", units);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
