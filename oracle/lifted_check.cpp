// oracle/lifted_check.cpp -- test infrastructure: the shim LiftedProblem's device mode (over
// gridnlp_b200::CudaOpfNlp) against the reference's own LiftedProblem (the shim's host mode,
// i.e. the unmodified reference class, over the reference's PatternNlp) on the same network:
// sizes, boxes, slack boxes (relative and absolute relaxation), lifted COO structures,
// free map, to_full, and the lifted evaluations at an interior point.  Prints one JSON line
// of mismatch counts (all zero when the shim is faithful) and the largest relative value
// difference of the evaluations (the callbacks' 1e-12 bar; structures and boxes bit-exact).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "gridnlp/ipm/lifted.hpp"  // resolves to the shim
#include "gridnlp/ipm/pattern_nlp.hpp"
#include "gridnlp/power/opf.hpp"
#include "gridnlp_b200/cuda_opf_nlp.hpp"
#include "netbin.hpp"

#ifndef GRIDNLP_B200_LIFTED_SHIM
#error "the shim lifted.hpp must shadow the reference header"
#endif

using namespace gridnlp;

template <class A, class B>
static long diff_exact(const A& a, const B& b) {
  if (a.size() != b.size()) return -1;
  long d = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const bool same = a[i] == b[i] || (std::isnan(static_cast<double>(a[i])) &&
                                       std::isnan(static_cast<double>(b[i])));
    if (!same) ++d;
  }
  return d;
}

static double rel_diff(std::span<const double> a, std::span<const double> b) {
  double worst = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double den = std::max(std::abs(b[i]), 1e-2);
    worst = std::max(worst, std::abs(a[i] - b[i]) / den);
  }
  return worst;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: lifted_check <network.bin>\n");
    return 2;
  }
  try {
    const power::MultiPeriodCase mpc = netbin::load(argv[1]);
    power::BuiltOpf built = power::build_multiperiod_opf(mpc);
    ipm::PatternNlp ref_nlp(built.model);
    gridnlp_b200::CudaOpfNlp cuda_nlp(mpc);
    std::printf("[");
    const struct { double relax; bool absolute; } cases[] = {{1e-4, false}, {1e-3, true}};
    bool first = true;
    for (const auto& cs : cases) {
      ipm::LiftedProblem host(ref_nlp, cs.relax, cs.absolute);   // the reference class
      ipm::LiftedProblem dev(cuda_nlp, cs.relax, cs.absolute);   // the device mode
      long d_struct = 0, d_boxes = 0;
      d_struct += dev.n() != host.n() || dev.m() != host.m();
      d_struct += diff_exact(dev.jac_rows(), host.jac_rows());
      d_struct += diff_exact(dev.jac_cols(), host.jac_cols());
      d_struct += diff_exact(dev.hess_rows(), host.hess_rows());
      d_struct += diff_exact(dev.hess_cols(), host.hess_cols());
      d_struct += diff_exact(dev.free_to_full(), host.free_to_full());
      d_boxes += diff_exact(dev.x_lower(), host.x_lower());
      d_boxes += diff_exact(dev.x_upper(), host.x_upper());
      d_boxes += diff_exact(dev.x_start(), host.x_start());
      d_boxes += diff_exact(dev.s_lower(), host.s_lower());
      d_boxes += diff_exact(dev.s_upper(), host.s_upper());
      // an interior point of the lifted boxes
      const size_t n = static_cast<size_t>(host.n()), m = static_cast<size_t>(host.m());
      std::mt19937_64 rng(7);
      std::uniform_real_distribution<double> u(0.0, 1.0);
      std::vector<double> x(n), w(m);
      const auto xl = host.x_lower(), xu = host.x_upper(), xs = host.x_start();
      for (size_t i = 0; i < n; ++i) {
        const bool box = std::isfinite(xl[i]) && std::isfinite(xu[i]);
        x[i] = box ? xl[i] + (0.15 + 0.7 * u(rng)) * (xu[i] - xl[i]) : xs[i] + 0.2 * (u(rng) - 0.5);
      }
      for (auto& v : w) v = 2.0 * u(rng) - 1.0;
      std::vector<double> fa(static_cast<size_t>(cuda_nlp.n_vars())),
          fb(static_cast<size_t>(cuda_nlp.n_vars()));
      dev.to_full(x, fa);
      host.to_full(x, fb);
      const long d_tofull = diff_exact(fa, fb);
      double f1 = 0, f2 = 0;
      std::vector<double> g1(n), g2(n), c1(m), c2(m);
      std::vector<double> j1(static_cast<size_t>(host.jac_nnz())), j2(j1.size());
      std::vector<double> h1(static_cast<size_t>(host.hess_nnz())), h2(h1.size());
      const bool ok = dev.eval_f(x, f1) && host.eval_f(x, f2) && dev.eval_grad(x, g1) &&
                      host.eval_grad(x, g2) && dev.eval_g(x, c1) && host.eval_g(x, c2) &&
                      dev.eval_jac(x, j1) && host.eval_jac(x, j2) &&
                      dev.eval_hess(x, w, 0.7, h1) && host.eval_hess(x, w, 0.7, h2);
      const double rf = std::abs(f1 - f2) / std::max(std::abs(f2), 1e-2);
      const double worst = std::max({rf, rel_diff(g1, g2), rel_diff(c1, c2), rel_diff(j1, j2),
                                     rel_diff(h1, h2)});
      std::printf("%s{\"relax\": %g, \"absolute\": %s, \"device_mode\": %d, \"host_mode\": %d, "
                  "\"n\": %zu, \"m\": %zu, \"struct_diff\": %ld, \"boxes_diff\": %ld, "
                  "\"to_full_diff\": %ld, \"evals_ok\": %d, \"grad_diff\": %ld, "
                  "\"max_rel_diff\": %.3e}",
                  first ? "" : ", ", cs.relax, cs.absolute ? "true" : "false",
                  dev.b200_device() ? 1 : 0, host.b200_device() ? 0 : 1, n, m, d_struct, d_boxes,
                  d_tofull, ok ? 1 : 0, diff_exact(g1, g2), worst);
      first = false;
    }
    std::printf("]\n");
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
