// include/gridnlp_b200/shim/gridnlp/ipm/condensed.hpp
//
// Drop-in #2: a replacement for the reference's concrete
// gridnlp::ipm::CondensedKkt (ipm/condensed.hpp:27-185), picked up by
// include-path shadowing — put  -I<repo>/include/gridnlp_b200/shim  BEFORE the
// reference include directory and the unmodified IpmSolver (ipm/solver.hpp:133-251)
// constructs this class instead.  Same public surface and semantics:
//   * constructor: CSR(A) + M = Hess U AtA U diag pattern built on the B200
//     (gn_kkt_create; for the lifted structure of a CudaOpfNlp the library recognises
//     the OPF problem and uses its specialised kernels); the reference's own LDL^T
//     symbolic phase runs on the host at the first factorize() / factor_nnz() (the
//     reference runs it in the ctor; the result is the same object);
//   * set_jacobian / assemble: the scatter and the condensed assembly run on the
//     GPU (bit-identical to the reference for equal inputs);
//   * factorize / solve stay on the reference's sparse::LdltSolver (out of scope
//     for the B200 path; "sparse factorization ... stays behind the reference's
//     linear-solver interface").
#pragma once

#include <algorithm>
#include <cstdlib>
#include <optional>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "gridnlp/common.hpp"
#include "gridnlp/ipm/iterate.hpp"
#include "gridnlp/sparse/ldlt.hpp"
#include "gridnlp/sparse/matrix.hpp"
#include "gridnlp_b200.h"

#define GRIDNLP_B200_CONDENSED_SHIM 1

namespace gridnlp::ipm {

// (not in the reference) KKTs built by this process: [generic, OPF-specialised]
inline long b200_kkt_counts[2] = {0, 0};

// (not in the reference) the A and M values the GPU returns every iteration, kept in
// page-locked memory (gn_host_alloc) so their device->host copies are direct DMA; plain
// heap memory when the pinned allocation fails (same values, slower copies).
class B200HostValues {
 public:
  B200HostValues() = default;
  explicit B200HostValues(size_t n) : n_(n) {
    void* p = nullptr;
    if (n && gn_host_alloc(n * sizeof(double), &p) == GN_OK && p) {
      p_ = static_cast<double*>(p);
      pinned_ = true;
    } else if (n) {
      p_ = new double[n];
    }
    std::fill(p_, p_ + n_, 0.0);
  }
  ~B200HostValues() { release(); }
  B200HostValues(const B200HostValues&) = delete;
  B200HostValues& operator=(const B200HostValues&) = delete;
  B200HostValues& operator=(B200HostValues&& o) noexcept {
    release();
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(pinned_, o.pinned_);
    return *this;
  }
  double* data() { return p_; }
  size_t size() const { return n_; }
  bool pinned() const { return pinned_; }
  operator std::span<const double>() const { return {p_, n_}; }

 private:
  void release() {
    if (pinned_) gn_host_free(p_);
    else delete[] p_;
    p_ = nullptr;
    n_ = 0;
    pinned_ = false;
  }
  double* p_ = nullptr;
  size_t n_ = 0;
  bool pinned_ = false;
};

class CondensedKkt {
 public:
  CondensedKkt(index_t n, index_t m, std::span<const index_t> jac_rows,
               std::span<const index_t> jac_cols, std::span<const index_t> hess_rows,
               std::span<const index_t> hess_cols, sparse::LdltOptions ldlt_opts = {})
      : n_(n), m_(m) {
    const char* dev = std::getenv("GRIDNLP_B200_DEVICE");
    gn_error err{};
    if (gn_kkt_create(n, m, static_cast<int64_t>(jac_rows.size()), jac_rows.data(),
                      jac_cols.data(), static_cast<int64_t>(hess_rows.size()), hess_rows.data(),
                      hess_cols.data(), dev ? std::atoi(dev) : 0, &kkt_, &err) != GN_OK)
      throw Error(std::string("CondensedKkt (gridnlp_b200): ") + err.message);
    int64_t dims[9] = {};
    gn_kkt_dims(kkt_, dims);
    a_.nrows = m;
    a_.ncols = n;
    a_.rowptr.resize(static_cast<size_t>(m) + 1);
    a_.colidx.resize(static_cast<size_t>(dims[1]));
    mpat_.nrows = mpat_.ncols = n;
    mpat_.colptr.resize(static_cast<size_t>(n) + 1);
    mpat_.rowidx.resize(static_cast<size_t>(dims[2]));
    gn_kkt_structure(kkt_, a_.rowptr.data(), a_.colidx.data(), mpat_.colptr.data(),
                     mpat_.rowidx.data(), GN_MEM_HOST);
    a_vals_ = B200HostValues(a_.colidx.size());
    mvals_ = B200HostValues(mpat_.rowidx.size());
    ldlt_opts_ = ldlt_opts;
    int64_t d2[9] = {};
    gn_kkt_dims(kkt_, d2);
    specialised_ = d2[7] == 1;
    ++b200_kkt_counts[specialised_ ? 1 : 0];
    cvec_.assign(static_cast<size_t>(m), 0.0);
    dvec_.assign(static_cast<size_t>(m), 0.0);
    sig_dw_.assign(static_cast<size_t>(m), 0.0);
    tm_.assign(static_cast<size_t>(m), 0.0);
    rhs_.assign(static_cast<size_t>(n), 0.0);
  }
  ~CondensedKkt() { gn_kkt_destroy(kkt_); }
  CondensedKkt(const CondensedKkt&) = delete;
  CondensedKkt& operator=(const CondensedKkt&) = delete;

  index_t dim() const { return n_; }
  const sparse::CsrPattern& jacobian_csr() const { return a_; }
  std::span<const double> jacobian_values() const {
    wait_a();
    return a_vals_;
  }
  const sparse::CscPattern& pattern() const { return mpat_; }
  std::span<const double> values() const { return mvals_; }
  index_t factor_nnz() const { return ldlt().factor_nnz(); }
  // (not in the reference) true when the OPF-specialised kernels assemble this KKT
  bool b200_specialised() const { return specialised_; }

  // A = scatter(J) on the GPU; the values come back for the host solves.  Into page-locked
  // memory the copy runs on a side stream while the IPM carries on (the next assemble's
  // uploads go the other way over PCIe); every reader of A waits for it first.
  void set_jacobian(std::span<const double> jac_vals) {
    wait_a();
    if (gn_kkt_set_jacobian(kkt_, jac_vals.data(), GN_MEM_HOST) != GN_OK)
      throw Error("CondensedKkt::set_jacobian (gridnlp_b200) failed");
    if (a_vals_.pinned()) {
      if (gn_kkt_values_start(kkt_, a_vals_.data(), nullptr) != GN_OK)
        throw Error("CondensedKkt::set_jacobian (gridnlp_b200) read-back failed");
      a_pending_ = true;
    } else if (gn_kkt_values(kkt_, a_vals_.data(), nullptr, GN_MEM_HOST) != GN_OK) {
      throw Error("CondensedKkt::set_jacobian (gridnlp_b200) failed");
    }
  }

  // M = W + dw I + Sx + At D A on the GPU; the per-row C/D factors the solve
  // needs are recomputed on the host with the same expressions.
  void assemble(std::span<const double> hess_vals, std::span<const double> sigma_x,
                std::span<const double> sigma_s, double delta_w, double delta_c) {
    delta_c_ = delta_c;
    // the GPU call (uploads, assembly, M back) runs beside the host's per-row factors
    int rc = GN_OK;
    std::thread gpu([&] {
      rc = gn_kkt_assemble(kkt_, hess_vals.data(), sigma_x.data(), sigma_s.data(), delta_w,
                           delta_c, GN_MEM_HOST);
      if (rc == GN_OK) rc = gn_kkt_values(kkt_, nullptr, mvals_.data(), GN_MEM_HOST);
    });
    for (index_t i = 0; i < m_; ++i) {
      const size_t u = static_cast<size_t>(i);
      const double sd = sigma_s[u] + delta_w;
      const double c = 1.0 / (1.0 + delta_c * sd);
      cvec_[u] = c;
      dvec_[u] = sd * c;
      sig_dw_[u] = sd;
    }
    gpu.join();
    if (rc != GN_OK) throw Error("CondensedKkt::assemble (gridnlp_b200) failed");
  }

  bool factorize() {
    ldlt().factorize(mvals_);
    const sparse::Inertia& in = ldlt().inertia();
    return in.positive == n_ && in.negative == 0 && in.zero == 0;
  }
  const sparse::Inertia& inertia() const { return ldlt().inertia(); }
  index_t floored_pivots() const { return ldlt().floored_pivots(); }

  // Reduced solve: M dx = -(qx + At (C qs + D qy)), ds = C (A dx + qy - dc qs),
  // dy = -qs - (Ss + dw) ds  (the class comment of condensed.hpp:17-26).
  double solve(std::span<const double> qx, std::span<const double> qs,
               std::span<const double> qy, Direction& d, int refine_passes) {
    wait_a();
    for (index_t i = 0; i < m_; ++i) {
      const size_t u = static_cast<size_t>(i);
      tm_[u] = cvec_[u] * qs[u] + dvec_[u] * qy[u];
    }
    sparse::csr_matvec_transpose(a_, a_vals_, tm_, rhs_);
    for (index_t i = 0; i < n_; ++i) {
      const size_t u = static_cast<size_t>(i);
      rhs_[u] = -(qx[u] + rhs_[u]);
    }
    d.dx.assign(static_cast<size_t>(n_), 0.0);
    d.ds.assign(static_cast<size_t>(m_), 0.0);
    d.dy.assign(static_cast<size_t>(m_), 0.0);
    ldlt().solve(rhs_, d.dx);
    const double resid = ldlt().refine(mvals_, rhs_, d.dx, refine_passes);
    sparse::csr_matvec(a_, a_vals_, d.dx, tm_);
    for (index_t i = 0; i < m_; ++i) {
      const size_t u = static_cast<size_t>(i);
      d.ds[u] = cvec_[u] * (tm_[u] + qy[u] - delta_c_ * qs[u]);
      d.dy[u] = -qs[u] - sig_dw_[u] * d.ds[u];
    }
    return resid;
  }

 private:
  void wait_a() const {
    if (!a_pending_) return;
    if (gn_kkt_values_wait(kkt_) != GN_OK) throw Error("CondensedKkt: A read-back failed");
    a_pending_ = false;
  }
  // the reference's LDL^T (AMD + symbolic analysis) on M's pattern, built once on first use
  sparse::LdltSolver& ldlt() const {
    if (!ldlt_) ldlt_.emplace(mpat_, std::vector<index_t>{}, ldlt_opts_);
    return *ldlt_;
  }

  gn_kkt* kkt_ = nullptr;
  bool specialised_ = false;
  sparse::LdltOptions ldlt_opts_{};
  index_t n_, m_;
  sparse::CsrPattern a_;
  B200HostValues a_vals_;
  mutable bool a_pending_ = false;  // A still on its way back (set_jacobian)
  sparse::CscPattern mpat_;
  B200HostValues mvals_;
  mutable std::optional<sparse::LdltSolver> ldlt_;
  std::vector<double> cvec_, dvec_, sig_dw_, tm_, rhs_;
  double delta_c_ = 0.0;
};

// Bound-multiplier steps from (dx, ds): for each present bound,
//   lower: dz = -(pz + z * dw) / (w - wl),   upper: dz = (-pz + z * dw) / (wu - w).
inline void recover_bound_steps(const Iterate& it, const Residuals& r,
                                std::span<const double> xl, std::span<const double> xu,
                                std::span<const double> sl, std::span<const double> su,
                                Direction& d) {
  auto side = [](std::span<const double> w, std::span<const double> dw,
                 std::span<const double> lo, std::span<const double> hi,
                 std::span<const double> zl, std::span<const double> zu,
                 std::span<const double> pzl, std::span<const double> pzu,
                 std::vector<double>& dzl, std::vector<double>& dzu) {
    const size_t k = w.size();
    dzl.assign(k, 0.0);
    dzu.assign(k, 0.0);
    for (size_t i = 0; i < k; ++i) {
      if (has_lower(lo[i])) dzl[i] = -(pzl[i] + zl[i] * dw[i]) / (w[i] - lo[i]);
      if (has_upper(hi[i])) dzu[i] = (-pzu[i] + zu[i] * dw[i]) / (hi[i] - w[i]);
    }
  };
  side(it.x, d.dx, xl, xu, it.zlx, it.zux, r.pzlx, r.pzux, d.dzlx, d.dzux);
  side(it.s, d.ds, sl, su, it.zls, it.zus, r.pzls, r.pzus, d.dzls, d.dzus);
}

}  // namespace gridnlp::ipm
