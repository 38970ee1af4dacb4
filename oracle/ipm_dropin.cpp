// oracle/ipm_dropin.cpp — end-to-end drop-in check (test infrastructure).
//
// Runs the UNMODIFIED reference interior-point driver (ipm::solve_nlp,
// ipm/solver.hpp:469) on the multi-period OPF with the B200 path plugged in
// through the reference's own seams:
//   --nlp cuda : gridnlp_b200::CudaOpfNlp (NlpProblem over the C-ABI)
//   --nlp ref  : the reference's PatternNlp (CPU tape callbacks)
// In both cases the condensed KKT is the shim CondensedKkt
// (include/gridnlp_b200/shim, found first on the include path), i.e. the B200
// set_jacobian/assemble feeding the reference LDL^T, and the lifted problem is the shim
// LiftedProblem (device gathers over CudaOpfNlp; the reference's own class over
// PatternNlp and the restoration problem).  Prints one JSON line.
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
#include "netbin.hpp"

#ifndef GRIDNLP_B200_CONDENSED_SHIM
#error "the shim condensed.hpp must shadow the reference header"
#endif
#ifndef GRIDNLP_B200_LIFTED_SHIM
#error "the shim lifted.hpp must shadow the reference header"
#endif

using namespace gridnlp;


int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: ipm_dropin <network.bin> cuda|ref [tol] [repeat]\n");
    return 2;
  }
  try {
    const power::MultiPeriodCase mpc = netbin::load(argv[1]);
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
                "\"kkt_generic\": %ld, \"kkt_specialised\": %ld, \"lifted_host\": %ld, "
                "\"lifted_device\": %ld}\n",
                which.c_str(), r.iterations, r.objective, ipm::to_string(r.status),
                r.restorations, secs, warm, ipm::b200_kkt_counts[0], ipm::b200_kkt_counts[1],
                ipm::b200_lifted_counts[0], ipm::b200_lifted_counts[1]);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
