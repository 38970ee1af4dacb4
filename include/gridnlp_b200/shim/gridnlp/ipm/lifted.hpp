// include/gridnlp_b200/shim/gridnlp/ipm/lifted.hpp
//
// Drop-in #3: a replacement for the reference's
// gridnlp::ipm::LiftedProblem (ipm/lifted.hpp:22-200), picked up by the same include-path
// shadowing as the CondensedKkt shim (-I<repo>/include/gridnlp_b200/shim before the
// reference include directory).  The unmodified IpmSolver (solver.hpp:97, 471-476) and
// RestorationNlp (restoration.hpp:24-184) drive it through the same members.
//
// Two modes, chosen in the constructor:
//   * device -- the wrapped problem is a gridnlp_b200::CudaOpfNlp: the fixed-variable
//     filter is the library's (gn_lifted_create, bit-identical COO and free map), and every
//     eval_* is ONE library call on the free-variable vector: staging into the full space,
//     the callback and the J / H value gathers all run on the B200, and only lifted-size
//     arrays cross PCIe.  The reference does the staging and the O(J + H) pick gathers on
//     the host per call (lifted.hpp:128-168), which is most of the seam's time at scale.
//   * host -- any other NlpProblem (the reference's PatternNlp, the restoration problem):
//     the reference's own class, included below under another name and used unchanged.
// GRIDNLP_B200_HOST_LIFTED=1 forces the host mode (for timing the two side by side).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <optional>
#include <span>
#include <vector>

#include "gridnlp/common.hpp"
#include "gridnlp/ipm/nlp.hpp"
#include "gridnlp_b200/cuda_opf_nlp.hpp"

// the reference's LiftedProblem, unmodified, as gridnlp::ipm::LiftedProblemHost
#define LiftedProblem LiftedProblemHost
#include_next <gridnlp/ipm/lifted.hpp>
#undef LiftedProblem

#define GRIDNLP_B200_LIFTED_SHIM 1

namespace gridnlp::ipm {

// (not in the reference) lifted problems built by this process: [host, device]
inline long b200_lifted_counts[2] = {0, 0};

class LiftedProblem {
 public:
  LiftedProblem(NlpProblem& nlp, double relax, bool absolute_relaxation = false)
      : nlp_(&nlp) {
    const char* env = std::getenv("GRIDNLP_B200_HOST_LIFTED");
    cuda_ = (env && env[0] == '1') ? nullptr : dynamic_cast<gridnlp_b200::CudaOpfNlp*>(&nlp);
    ++b200_lifted_counts[cuda_ ? 1 : 0];
    if (!cuda_) {
      host_.emplace(nlp, relax, absolute_relaxation);
      return;
    }
    auto L = cuda_->lift(relax);
    free_to_full_ = std::move(L.free_to_full);
    jac_rows_ = std::move(L.jac_rows);
    jac_cols_ = std::move(L.jac_cols);
    hess_rows_ = std::move(L.hess_rows);
    hess_cols_ = std::move(L.hess_cols);
    // boxes of the free variables; the pinned values of the fixed ones (for to_full)
    const auto xl = nlp.x_lower(), xu = nlp.x_upper(), xs = nlp.x_start();
    pinned_.resize(xl.size());
    for (size_t i = 0; i < xl.size(); ++i) pinned_[i] = xl[i] == xu[i] ? xl[i] : 0.0;
    const size_t n = free_to_full_.size();
    x_lower_.resize(n);
    x_upper_.resize(n);
    x_start_.resize(n);
    for (size_t k = 0; k < n; ++k) {
      const size_t i = static_cast<size_t>(free_to_full_[k]);
      x_lower_[k] = xl[i];
      x_upper_[k] = xu[i];
      x_start_[k] = xs[i];
    }
    // slack boxes: equality rows get the relaxation box (lifted.hpp:48-65 semantics)
    const auto rl = nlp.row_lower(), ru = nlp.row_upper();
    s_lower_.assign(rl.begin(), rl.end());
    s_upper_.assign(ru.begin(), ru.end());
    for (size_t i = 0; i < rl.size(); ++i) {
      if (rl[i] != ru[i]) continue;
      const double half = absolute_relaxation ? relax : relax * std::max(1.0, std::abs(rl[i]));
      s_lower_[i] = rl[i] - half;
      s_upper_[i] = ru[i] + half;
    }
  }

  NlpProblem& inner() { return *nlp_; }
  index_t n() const { return host_ ? host_->n() : static_cast<index_t>(free_to_full_.size()); }
  index_t m() const { return nlp_->n_cons(); }

  std::span<const double> x_lower() const { return host_ ? host_->x_lower() : x_lower_; }
  std::span<const double> x_upper() const { return host_ ? host_->x_upper() : x_upper_; }
  std::span<const double> x_start() const { return host_ ? host_->x_start() : x_start_; }
  std::span<const double> s_lower() const { return host_ ? host_->s_lower() : s_lower_; }
  std::span<const double> s_upper() const { return host_ ? host_->s_upper() : s_upper_; }

  std::span<const index_t> jac_rows() const { return host_ ? host_->jac_rows() : jac_rows_; }
  std::span<const index_t> jac_cols() const { return host_ ? host_->jac_cols() : jac_cols_; }
  std::span<const index_t> hess_rows() const { return host_ ? host_->hess_rows() : hess_rows_; }
  std::span<const index_t> hess_cols() const { return host_ ? host_->hess_cols() : hess_cols_; }
  index_t jac_nnz() const { return static_cast<index_t>(jac_rows().size()); }
  index_t hess_nnz() const { return static_cast<index_t>(hess_rows().size()); }

  void to_full(std::span<const double> x, std::span<double> out) const {
    if (host_) return host_->to_full(x, out);
    std::copy(pinned_.begin(), pinned_.end(), out.begin());
    for (size_t k = 0; k < free_to_full_.size(); ++k)
      out[static_cast<size_t>(free_to_full_[k])] = x[k];
  }
  std::span<const index_t> free_to_full() const {
    return host_ ? host_->free_to_full() : std::span<const index_t>(free_to_full_);
  }

  bool eval_f(std::span<const double> x, double& out) {
    return host_ ? host_->eval_f(x, out) : cuda_->lifted_eval_f(x, out);
  }
  bool eval_g(std::span<const double> x, std::span<double> out) {
    return host_ ? host_->eval_g(x, out) : cuda_->lifted_eval_g(x, out);
  }
  bool eval_grad(std::span<const double> x, std::span<double> out) {
    return host_ ? host_->eval_grad(x, out) : cuda_->lifted_eval_grad(x, out);
  }
  bool eval_jac(std::span<const double> x, std::span<double> out) {
    return host_ ? host_->eval_jac(x, out) : cuda_->lifted_eval_jac(x, out);
  }
  bool eval_hess(std::span<const double> x, std::span<const double> row_weights,
                 double obj_weight, std::span<double> out) {
    return host_ ? host_->eval_hess(x, row_weights, obj_weight, out)
                 : cuda_->lifted_eval_hess(x, row_weights, obj_weight, out);
  }

  // (not in the reference) true when the evaluations run through the library's lifted calls
  bool b200_device() const { return cuda_ != nullptr; }

 private:
  NlpProblem* nlp_;
  gridnlp_b200::CudaOpfNlp* cuda_ = nullptr;
  std::optional<LiftedProblemHost> host_;
  // device mode
  std::vector<index_t> free_to_full_, jac_rows_, jac_cols_, hess_rows_, hess_cols_;
  std::vector<double> pinned_, x_lower_, x_upper_, x_start_, s_lower_, s_upper_;
};

}  // namespace gridnlp::ipm
