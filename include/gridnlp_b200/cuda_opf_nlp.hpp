// include/gridnlp_b200/cuda_opf_nlp.hpp — the reference's NlpProblem plugin
// interface backed by the B200 C-ABI.
//
// Drop-in #1: gridnlp::ipm::NlpProblem (ipm/nlp.hpp:15-39) is the
// reference's only virtual callback boundary.  CudaOpfNlp implements it for the
// multi-period AC-OPF that power::build_multiperiod_opf + ipm::PatternNlp
// (power/opf.hpp:100, ipm/pattern_nlp.hpp:15-62) expose, evaluating every
// callback with the sm_100a kernels of libgridnlp_b200.so.  Same sizes, bounds,
// COO structures (bit-identical) and the same error behaviour: shape mistakes
// throw gridnlp::Error, evaluation failures return false and are described by
// last_failure().  Header-only; include it with the reference's include path and
// link libgridnlp_b200.so.
#pragma once

#include <cmath>
#include <span>
#include <string>
#include <vector>

#include "gridnlp/common.hpp"
#include "gridnlp/ipm/nlp.hpp"
#include "gridnlp/power/network.hpp"
#include "gridnlp_b200.h"

namespace gridnlp_b200 {

class CudaOpfNlp final : public gridnlp::ipm::NlpProblem {
 public:
  // Equivalent of build_multiperiod_opf(mpc) + PatternNlp on device `device`.
  explicit CudaOpfNlp(const gridnlp::power::MultiPeriodCase& mpc, int device = 0) {
    const auto& net = mpc.network;
    const gridnlp::index_t N = net.n_buses(), L = net.n_lines(), G = net.n_generators(),
                           D = net.n_loads();
    if (mpc.profile.n_loads != D)
      throw gridnlp::Error("opf: load profile does not match network loads");
    for (const auto& b : net.buses) {
      bus_vmin_.push_back(b.v_min);
      bus_vmax_.push_back(b.v_max);
    }
    for (const auto& l : net.lines) {
      lf_.push_back(l.from);
      lt_.push_back(l.to);
      lg_.push_back(l.g);
      lb_.push_back(l.b);
      ls_.push_back(l.s_max);
      la_.push_back(l.angle_min);
      lA_.push_back(l.angle_max);
    }
    for (const auto& g : net.generators) {
      gb_.push_back(g.bus);
      gpmin_.push_back(g.p_min);
      gpmax_.push_back(g.p_max);
      gqmin_.push_back(g.q_min);
      gqmax_.push_back(g.q_max);
      gramp_.push_back(g.ramp);
      gc2_.push_back(g.c2);
      gc1_.push_back(g.c1);
      gc0_.push_back(g.c0);
      gps_.push_back(g.p_start);
      gqs_.push_back(g.q_start);
    }
    for (const auto& d : net.loads) {
      db_.push_back(d.bus);
      dp_.push_back(d.p);
      dq_.push_back(d.q);
    }
    gn_network c{};
    c.n_bus = N;
    c.n_line = L;
    c.n_gen = G;
    c.n_load = D;
    c.reference_bus = net.reference_bus;
    c.bus_vmin = bus_vmin_.data();
    c.bus_vmax = bus_vmax_.data();
    c.vm_start = net.vm_start.data();
    c.va_start = net.va_start.data();
    c.line_from = lf_.data();
    c.line_to = lt_.data();
    c.line_g = lg_.data();
    c.line_b = lb_.data();
    c.line_smax = ls_.data();
    c.line_amin = la_.data();
    c.line_amax = lA_.data();
    c.gen_bus = gb_.data();
    c.gen_pmin = gpmin_.data();
    c.gen_pmax = gpmax_.data();
    c.gen_qmin = gqmin_.data();
    c.gen_qmax = gqmax_.data();
    c.gen_ramp = gramp_.data();
    c.gen_c2 = gc2_.data();
    c.gen_c1 = gc1_.data();
    c.gen_c0 = gc0_.data();
    c.gen_pstart = gps_.data();
    c.gen_qstart = gqs_.data();
    c.load_bus = db_.data();
    c.load_p = dp_.data();
    c.load_q = dq_.data();
    gn_error err{};
    if (gn_ctx_create(&c, mpc.periods(), mpc.profile.scale.data(), device, &ctx_, &err) != GN_OK)
      throw gridnlp::Error(std::string("gn_ctx_create: ") + err.message);
    gn_sizes s{};
    gn_ctx_sizes(ctx_, &s);
    n_ = static_cast<gridnlp::index_t>(s.n_vars);
    m_ = static_cast<gridnlp::index_t>(s.n_cons);
    xl_.resize(n_);
    xu_.resize(n_);
    xs_.resize(n_);
    rl_.resize(m_);
    ru_.resize(m_);
    gn_ctx_bounds(ctx_, xl_.data(), xu_.data(), xs_.data(), rl_.data(), ru_.data());
    jr_.resize(s.jac_nnz);
    jc_.resize(s.jac_nnz);
    hr_.resize(s.hess_nnz);
    hc_.resize(s.hess_nnz);
    gn_jac_structure(ctx_, jr_.data(), jc_.data(), GN_MEM_HOST);
    gn_hess_structure(ctx_, hr_.data(), hc_.data(), GN_MEM_HOST);
    // the CondensedKkt the IpmSolver builds from this problem's lifted COO (solver.hpp:
    // 139-141) is recognised by the library and gets the OPF-specialised assembly
    if (gn_ctx_publish(ctx_, 1) != GN_OK) throw gridnlp::Error("gn_ctx_publish failed");
  }
  ~CudaOpfNlp() override { gn_ctx_destroy(ctx_); }
  CudaOpfNlp(const CudaOpfNlp&) = delete;
  CudaOpfNlp& operator=(const CudaOpfNlp&) = delete;

  gridnlp::index_t n_vars() const override { return n_; }
  gridnlp::index_t n_cons() const override { return m_; }
  std::span<const double> x_lower() const override { return xl_; }
  std::span<const double> x_upper() const override { return xu_; }
  std::span<const double> x_start() const override { return xs_; }
  std::span<const double> row_lower() const override { return rl_; }
  std::span<const double> row_upper() const override { return ru_; }
  std::span<const gridnlp::index_t> jac_rows() const override { return jr_; }
  std::span<const gridnlp::index_t> jac_cols() const override { return jc_; }
  std::span<const gridnlp::index_t> hess_rows() const override { return hr_; }
  std::span<const gridnlp::index_t> hess_cols() const override { return hc_; }

  bool eval_f(std::span<const double> x, double& out) override {
    check(x.size(), n_, "eval_f: bad x size");
    return record(gn_eval_f(ctx_, x.data(), &out, GN_MEM_HOST, &err_));
  }
  bool eval_grad(std::span<const double> x, std::span<double> out) override {
    check(x.size(), n_, "eval_grad: bad x size");
    check(out.size(), n_, "eval_grad: bad output size");
    return record(gn_eval_grad(ctx_, x.data(), out.data(), GN_MEM_HOST, &err_));
  }
  bool eval_g(std::span<const double> x, std::span<double> out) override {
    check(x.size(), n_, "eval_g: bad x size");
    check(out.size(), m_, "eval_g: bad output size");
    return record(gn_eval_g(ctx_, x.data(), out.data(), GN_MEM_HOST, &err_));
  }
  bool eval_jac(std::span<const double> x, std::span<double> out) override {
    check(x.size(), n_, "eval_jac: bad x size");
    check(out.size(), jr_.size(), "eval_jac: bad output size");
    return record(gn_eval_jac(ctx_, x.data(), out.data(), GN_MEM_HOST, &err_));
  }
  bool eval_hess(std::span<const double> x, std::span<const double> w, double ow,
                 std::span<double> out) override {
    check(x.size(), n_, "eval_hess: bad x size");
    check(w.size(), m_, "eval_hess: bad weight size");
    check(out.size(), hr_.size(), "eval_hess: bad output size");
    return record(gn_eval_hess(ctx_, x.data(), w.data(), ow, out.data(), GN_MEM_HOST, &err_));
  }

  // ---- the lifted problem on the device, for the shim ipm::LiftedProblem
  // (shim/gridnlp/ipm/lifted.hpp): the fixed-variable filter of lifted.hpp:25-100 is
  // built by the library; x is the free-variable vector and J / H come back lifted.
  struct Lifted {
    std::vector<gridnlp::index_t> free_to_full, jac_rows, jac_cols, hess_rows, hess_cols;
  };
  Lifted lift(double relax) {
    gn_error err{};
    if (gn_lifted_create(ctx_, relax, &err) != GN_OK)
      throw gridnlp::Error(std::string("gn_lifted_create: ") + err.message);
    gn_sizes s{};
    gn_ctx_sizes(ctx_, &s);
    nf_ = static_cast<size_t>(s.n_free);
    njl_ = static_cast<size_t>(s.jac_nnz_lifted);
    nhl_ = static_cast<size_t>(s.hess_nnz_lifted);
    Lifted L;
    L.free_to_full.resize(nf_);
    L.jac_rows.resize(njl_);
    L.jac_cols.resize(njl_);
    L.hess_rows.resize(nhl_);
    L.hess_cols.resize(nhl_);
    if (gn_lifted_structure(ctx_, L.free_to_full.data(), L.jac_rows.data(), L.jac_cols.data(),
                            nullptr, L.hess_rows.data(), L.hess_cols.data(), nullptr, nullptr,
                            nullptr, GN_MEM_HOST) != GN_OK)
      throw gridnlp::Error("gn_lifted_structure failed");
    return L;
  }
  bool lifted_eval_f(std::span<const double> x, double& out) {
    check(x.size(), nf_, "lifted eval_f: bad x size");
    return record(gn_lifted_eval_f(ctx_, x.data(), &out, GN_MEM_HOST, &err_));
  }
  bool lifted_eval_grad(std::span<const double> x, std::span<double> out) {
    check(x.size(), nf_, "lifted eval_grad: bad x size");
    check(out.size(), nf_, "lifted eval_grad: bad output size");
    return record(gn_lifted_eval_grad(ctx_, x.data(), out.data(), GN_MEM_HOST, &err_));
  }
  bool lifted_eval_g(std::span<const double> x, std::span<double> out) {
    check(x.size(), nf_, "lifted eval_g: bad x size");
    check(out.size(), m_, "lifted eval_g: bad output size");
    return record(gn_lifted_eval_g(ctx_, x.data(), out.data(), GN_MEM_HOST, &err_));
  }
  bool lifted_eval_jac(std::span<const double> x, std::span<double> out) {
    check(x.size(), nf_, "lifted eval_jac: bad x size");
    check(out.size(), njl_, "lifted eval_jac: bad output size");
    return record(gn_lifted_eval_jac(ctx_, x.data(), out.data(), GN_MEM_HOST, &err_));
  }
  bool lifted_eval_hess(std::span<const double> x, std::span<const double> w, double ow,
                        std::span<double> out) {
    check(x.size(), nf_, "lifted eval_hess: bad x size");
    check(w.size(), m_, "lifted eval_hess: bad weight size");
    check(out.size(), nhl_, "lifted eval_hess: bad output size");
    return record(gn_lifted_eval_hess(ctx_, x.data(), w.data(), ow, out.data(), GN_MEM_HOST,
                                      &err_));
  }

  // Diagnostic for the most recent failed evaluation (pattern_nlp.hpp:51-58).
  const std::string& last_failure() const { return last_failure_; }
  int last_failure_pattern() const { return err_.pattern; }
  int last_failure_record() const { return err_.record; }
  gn_ctx* context() { return ctx_; }

 private:
  static void check(size_t got, size_t want, const char* what) {
    if (got != want) throw gridnlp::Error(what);
  }
  bool record(int rc) {
    if (rc == GN_OK) return true;
    if (rc == GN_ERR_EVAL) {
      last_failure_ = err_.message;
      return false;
    }
    throw gridnlp::Error(std::string("gridnlp_b200: ") + err_.message);
  }

  gn_ctx* ctx_ = nullptr;
  gn_error err_{};
  gridnlp::index_t n_ = 0, m_ = 0;
  size_t nf_ = 0, njl_ = 0, nhl_ = 0;  // lifted sizes (after lift())
  std::vector<double> xl_, xu_, xs_, rl_, ru_;
  std::vector<gridnlp::index_t> jr_, jc_, hr_, hc_;
  std::vector<double> bus_vmin_, bus_vmax_, lg_, lb_, ls_, la_, lA_;
  std::vector<gridnlp::index_t> lf_, lt_, gb_, db_;
  std::vector<double> gpmin_, gpmax_, gqmin_, gqmax_, gramp_, gc2_, gc1_, gc0_, gps_, gqs_, dp_, dq_;
  std::string last_failure_;
};

}  // namespace gridnlp_b200
