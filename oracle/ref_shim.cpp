// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A thin extern "C" surface over the UNMODIFIED reference library
// (`gridnlp`, header-only C++20 under /root/reference/proj/include), compiled
// by oracle/Makefile into oracle/_ref/libgridnlp_ref.so.  Only tests/, the
// cpu_baseline leg of bench.py and `bench.py --impl reference` load it.  It
// contains no algorithm of its own: every entry point forwards to the
// reference's public API:
//   parse_matpower            power/matpower.hpp:119
//   build_multiperiod_opf     power/opf.hpp:100
//   PatternModel::evaluate_*  model/pattern_model.hpp:278-436 (+ set_threads :273)
//   LiftedProblem             ipm/lifted.hpp:25-100, 128-159
//   CondensedKkt              ipm/condensed.hpp:29-135
//   compress_to_csc           sparse/matrix.hpp:45
//   solve_nlp                 ipm/solver.hpp:469
//   iterate.hpp vector ops    ipm/iterate.hpp:42-298 (residuals, condensation,
//                             fraction to boundary, barrier, kkt_error), and
//                             recover_bound_steps, condensed.hpp:187-212
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "gridnlp/ipm/condensed.hpp"
#include "gridnlp/ipm/lifted.hpp"
#include "gridnlp/ipm/pattern_nlp.hpp"
#include "gridnlp/ipm/solver.hpp"
#include "gridnlp/power/matpower.hpp"
#include "gridnlp/power/network.hpp"
#include "gridnlp/power/opf.hpp"
#include "gridnlp/sparse/matrix.hpp"

using namespace gridnlp;

namespace {

void set_err(char* err, int len, const std::string& what) {
  if (!err || len <= 0) return;
  std::snprintf(err, static_cast<size_t>(len), "%s", what.c_str());
}

struct RefModel {
  power::MultiPeriodCase mpc;
  power::BuiltOpf built;
  std::unique_ptr<ipm::PatternNlp> nlp;
  std::unique_ptr<ipm::LiftedProblem> lifted;
  std::unique_ptr<ipm::CondensedKkt> kkt;
};

}  // namespace

extern "C" {

// ---------------------------------------------------------------- network
void* gnr_net_parse(const char* text, double ramp_fraction, char* err, int errlen) {
  try {
    power::MatpowerOptions opt;
    opt.ramp_fraction = ramp_fraction;
    return new power::NetworkData(power::parse_matpower(text, opt));
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void gnr_net_free(void* h) { delete static_cast<power::NetworkData*>(h); }

// dims: [n_bus, n_line, n_gen, n_load, reference_bus]
void gnr_net_dims(void* h, int32_t* dims) {
  auto* n = static_cast<power::NetworkData*>(h);
  dims[0] = n->n_buses();
  dims[1] = n->n_lines();
  dims[2] = n->n_generators();
  dims[3] = n->n_loads();
  dims[4] = n->reference_bus;
}

// Export the parsed per-unit data as SoA arrays (caller allocates).
void gnr_net_export(void* h, double* base_mva, double* bus_vmin, double* bus_vmax,
                    double* vm_start, double* va_start, int32_t* line_from,
                    int32_t* line_to, double* line_g, double* line_b, double* line_smax,
                    double* line_amin, double* line_amax, int32_t* gen_bus,
                    double* gen_pmin, double* gen_pmax, double* gen_qmin,
                    double* gen_qmax, double* gen_ramp, double* gen_c2, double* gen_c1,
                    double* gen_c0, double* gen_pstart, double* gen_qstart,
                    int32_t* load_bus, double* load_p, double* load_q) {
  auto* n = static_cast<power::NetworkData*>(h);
  *base_mva = n->base_mva;
  for (index_t i = 0; i < n->n_buses(); ++i) {
    bus_vmin[i] = n->buses[i].v_min;
    bus_vmax[i] = n->buses[i].v_max;
    vm_start[i] = n->vm_start[i];
    va_start[i] = n->va_start[i];
  }
  for (index_t l = 0; l < n->n_lines(); ++l) {
    const auto& L = n->lines[l];
    line_from[l] = L.from;
    line_to[l] = L.to;
    line_g[l] = L.g;
    line_b[l] = L.b;
    line_smax[l] = L.s_max;
    line_amin[l] = L.angle_min;
    line_amax[l] = L.angle_max;
  }
  for (index_t g = 0; g < n->n_generators(); ++g) {
    const auto& G = n->generators[g];
    gen_bus[g] = G.bus;
    gen_pmin[g] = G.p_min;
    gen_pmax[g] = G.p_max;
    gen_qmin[g] = G.q_min;
    gen_qmax[g] = G.q_max;
    gen_ramp[g] = G.ramp;
    gen_c2[g] = G.c2;
    gen_c1[g] = G.c1;
    gen_c0[g] = G.c0;
    gen_pstart[g] = G.p_start;
    gen_qstart[g] = G.q_start;
  }
  for (index_t j = 0; j < n->n_loads(); ++j) {
    load_bus[j] = n->loads[j].bus;
    load_p[j] = n->loads[j].p;
    load_q[j] = n->loads[j].q;
  }
}

// Reference load profile (network.hpp:104-140); scale is T x n_loads.
void gnr_load_profile(void* h, int32_t T, double resolution, uint64_t seed,
                      double amplitude, double noise, double* scale) {
  auto* n = static_cast<power::NetworkData*>(h);
  power::LoadProfile p =
      power::generate_load_profile(*n, T, resolution, seed, amplitude, noise);
  std::memcpy(scale, p.scale.data(), p.scale.size() * sizeof(double));
}

// ---------------------------------------------------------------- model
// Builds the reference multi-period OPF from a parsed network and an explicit
// T x n_loads scale table (so both arms see bit-identical demand).
void* gnr_model_create(void* h, int32_t T, const double* scale, char* err, int errlen) {
  try {
    auto* n = static_cast<power::NetworkData*>(h);
    auto m = std::make_unique<RefModel>();
    m->mpc.network = *n;
    m->mpc.profile.periods = T;
    m->mpc.profile.n_loads = n->n_loads();
    m->mpc.profile.scale.assign(scale, scale + static_cast<size_t>(T) * n->n_loads());
    m->built = power::build_multiperiod_opf(m->mpc);
    m->nlp = std::make_unique<ipm::PatternNlp>(m->built.model);
    return m.release();
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void gnr_model_free(void* h) { delete static_cast<RefModel*>(h); }

void gnr_model_set_threads(void* h, int n) {
  static_cast<RefModel*>(h)->built.model.set_threads(n);
}

// sizes: [n, m, jnnz, hnnz, n_thermal, n_ramp_gens]
void gnr_model_sizes(void* h, int64_t* s) {
  auto* m = static_cast<RefModel*>(h);
  s[0] = m->built.model.n_vars();
  s[1] = m->built.model.n_cons();
  s[2] = m->built.model.jac_nnz();
  s[3] = m->built.model.hess_nnz();
  s[4] = static_cast<int64_t>(m->built.layout.thermal_lines.size());
  s[5] = static_cast<int64_t>(m->built.layout.ramp_gens.size());
}

void gnr_model_bounds(void* h, double* xl, double* xu, double* xs, double* rl, double* ru) {
  auto* m = static_cast<RefModel*>(h);
  auto cp = [](std::span<const double> s, double* o) {
    std::memcpy(o, s.data(), s.size() * sizeof(double));
  };
  cp(m->built.model.x_lower(), xl);
  cp(m->built.model.x_upper(), xu);
  cp(m->built.model.x_start(), xs);
  cp(m->built.model.row_lower(), rl);
  cp(m->built.model.row_upper(), ru);
}

void gnr_model_structure(void* h, int32_t* jr, int32_t* jc, int32_t* hr, int32_t* hc) {
  auto* m = static_cast<RefModel*>(h);
  auto cp = [](std::span<const index_t> s, int32_t* o) {
    std::memcpy(o, s.data(), s.size() * sizeof(int32_t));
  };
  cp(m->built.model.jacobian_rows(), jr);
  cp(m->built.model.jacobian_cols(), jc);
  cp(m->built.model.hessian_rows(), hr);
  cp(m->built.model.hessian_cols(), hc);
}

// Evaluation status: returns 1 on success; on failure fills fail[0..1] =
// (pattern, record) from the reference EvalStatus (pattern_model.hpp:16-25).
static int status_out(const model::EvalStatus& st, int32_t* fail) {
  if (fail) {
    fail[0] = st.pattern;
    fail[1] = st.record;
  }
  return st.ok ? 1 : 0;
}

int gnr_eval_f(void* h, const double* x, double* out, int32_t* fail) {
  auto* m = static_cast<RefModel*>(h);
  const size_t n = static_cast<size_t>(m->built.model.n_vars());
  return status_out(m->built.model.evaluate_objective({x, n}, *out), fail);
}
int gnr_eval_grad(void* h, const double* x, double* out, int32_t* fail) {
  auto* m = static_cast<RefModel*>(h);
  const size_t n = static_cast<size_t>(m->built.model.n_vars());
  return status_out(m->built.model.evaluate_gradient({x, n}, {out, n}), fail);
}
int gnr_eval_g(void* h, const double* x, double* out, int32_t* fail) {
  auto* m = static_cast<RefModel*>(h);
  const size_t n = static_cast<size_t>(m->built.model.n_vars());
  const size_t mm = static_cast<size_t>(m->built.model.n_cons());
  return status_out(m->built.model.evaluate_constraints({x, n}, {out, mm}), fail);
}
int gnr_eval_jac(void* h, const double* x, double* out, int32_t* fail) {
  auto* m = static_cast<RefModel*>(h);
  const size_t n = static_cast<size_t>(m->built.model.n_vars());
  const size_t nj = static_cast<size_t>(m->built.model.jac_nnz());
  return status_out(m->built.model.evaluate_jacobian({x, n}, {out, nj}), fail);
}
int gnr_eval_hess(void* h, const double* x, const double* w, double ow, double* out,
                  int32_t* fail) {
  auto* m = static_cast<RefModel*>(h);
  const size_t n = static_cast<size_t>(m->built.model.n_vars());
  const size_t mm = static_cast<size_t>(m->built.model.n_cons());
  const size_t nh = static_cast<size_t>(m->built.model.hess_nnz());
  return status_out(
      m->built.model.evaluate_hessian({x, n}, {w, mm}, ow, {out, nh}), fail);
}

// ---------------------------------------------------------------- lifted
// sizes: [n_free, m, jnnz_lifted, hnnz_lifted]
void gnr_lifted_create(void* h, double relax, int64_t* sizes) {
  auto* m = static_cast<RefModel*>(h);
  m->lifted = std::make_unique<ipm::LiftedProblem>(*m->nlp, relax);
  sizes[0] = m->lifted->n();
  sizes[1] = m->lifted->m();
  sizes[2] = m->lifted->jac_nnz();
  sizes[3] = m->lifted->hess_nnz();
}

void gnr_lifted_structure(void* h, int32_t* free_to_full, int32_t* jr, int32_t* jc,
                          int32_t* hr, int32_t* hc, double* sl, double* su) {
  auto* m = static_cast<RefModel*>(h);
  auto cpi = [](std::span<const index_t> s, int32_t* o) {
    std::memcpy(o, s.data(), s.size() * sizeof(int32_t));
  };
  auto cpd = [](std::span<const double> s, double* o) {
    std::memcpy(o, s.data(), s.size() * sizeof(double));
  };
  cpi(m->lifted->free_to_full(), free_to_full);
  cpi(m->lifted->jac_rows(), jr);
  cpi(m->lifted->jac_cols(), jc);
  cpi(m->lifted->hess_rows(), hr);
  cpi(m->lifted->hess_cols(), hc);
  cpd(m->lifted->s_lower(), sl);
  cpd(m->lifted->s_upper(), su);
}

int gnr_lifted_eval_jac(void* h, const double* xfree, double* out) {
  auto* m = static_cast<RefModel*>(h);
  const size_t n = static_cast<size_t>(m->lifted->n());
  const size_t nj = static_cast<size_t>(m->lifted->jac_nnz());
  return m->lifted->eval_jac({xfree, n}, {out, nj}) ? 1 : 0;
}
int gnr_lifted_eval_hess(void* h, const double* xfree, const double* w, double ow,
                         double* out) {
  auto* m = static_cast<RefModel*>(h);
  const size_t n = static_cast<size_t>(m->lifted->n());
  const size_t mm = static_cast<size_t>(m->lifted->m());
  const size_t nh = static_cast<size_t>(m->lifted->hess_nnz());
  return m->lifted->eval_hess({xfree, n}, {w, mm}, ow, {out, nh}) ? 1 : 0;
}

// ---------------------------------------------------------------- condensed KKT
// sizes: [dim, a_nnz, m_nnz, factor_nnz]
void gnr_kkt_create(void* h, int64_t* sizes) {
  auto* m = static_cast<RefModel*>(h);
  auto& L = *m->lifted;
  m->kkt = std::make_unique<ipm::CondensedKkt>(L.n(), L.m(), L.jac_rows(), L.jac_cols(),
                                               L.hess_rows(), L.hess_cols());
  sizes[0] = m->kkt->dim();
  sizes[1] = m->kkt->jacobian_csr().nnz();
  sizes[2] = m->kkt->pattern().nnz();
  sizes[3] = m->kkt->factor_nnz();
}

void gnr_kkt_structure(void* h, int32_t* rowptr, int32_t* colidx, int32_t* colptr,
                       int32_t* rowidx) {
  auto* m = static_cast<RefModel*>(h);
  const auto& a = m->kkt->jacobian_csr();
  const auto& p = m->kkt->pattern();
  std::memcpy(rowptr, a.rowptr.data(), a.rowptr.size() * sizeof(int32_t));
  std::memcpy(colidx, a.colidx.data(), a.colidx.size() * sizeof(int32_t));
  std::memcpy(colptr, p.colptr.data(), p.colptr.size() * sizeof(int32_t));
  std::memcpy(rowidx, p.rowidx.data(), p.rowidx.size() * sizeof(int32_t));
}

void gnr_kkt_set_jacobian(void* h, const double* jvals_lifted) {
  auto* m = static_cast<RefModel*>(h);
  m->kkt->set_jacobian({jvals_lifted, static_cast<size_t>(m->lifted->jac_nnz())});
}

void gnr_kkt_assemble(void* h, const double* hvals_lifted, const double* sx,
                      const double* ss, double dw, double dc) {
  auto* m = static_cast<RefModel*>(h);
  m->kkt->assemble({hvals_lifted, static_cast<size_t>(m->lifted->hess_nnz())},
                   {sx, static_cast<size_t>(m->lifted->n())},
                   {ss, static_cast<size_t>(m->lifted->m())}, dw, dc);
}

void gnr_kkt_values(void* h, double* a_vals, double* m_vals) {
  auto* m = static_cast<RefModel*>(h);
  auto a = m->kkt->jacobian_values();
  auto v = m->kkt->values();
  if (a_vals) std::memcpy(a_vals, a.data(), a.size() * sizeof(double));
  if (m_vals) std::memcpy(m_vals, v.data(), v.size() * sizeof(double));
}

// ---------------------------------------------------------------- sparse KAT
// compress_to_csc on an arbitrary COO (matrix.hpp:45-81).
int gnr_compress_to_csc(int32_t nrows, int32_t ncols, int64_t nnz, const int32_t* rows,
                        const int32_t* cols, int32_t* colptr, int32_t* rowidx,
                        int32_t* slot_map) {
  sparse::CooPattern coo;
  coo.nrows = nrows;
  coo.ncols = ncols;
  coo.rows.assign(rows, rows + nnz);
  coo.cols.assign(cols, cols + nnz);
  std::vector<index_t> slots;
  sparse::CscPattern csc = sparse::compress_to_csc(coo, slots);
  std::memcpy(colptr, csc.colptr.data(), csc.colptr.size() * sizeof(int32_t));
  std::memcpy(rowidx, csc.rowidx.data(), csc.rowidx.size() * sizeof(int32_t));
  std::memcpy(slot_map, slots.data(), slots.size() * sizeof(int32_t));
  return csc.nnz();
}

// ---------------------------------------------------------------- end to end
// solve_nlp on the reference model (solver.hpp:469).  out: [iterations,
// objective, status, restorations, wall seconds of solve_nlp]
void gnr_solve(void* h, double tol, int max_iter, double* out) {
  auto* m = static_cast<RefModel*>(h);
  ipm::SolverConfig cfg;
  cfg.tol = tol;
  cfg.max_iter = max_iter;
  const auto t0 = std::chrono::steady_clock::now();
  ipm::SolveResult r = ipm::solve_nlp(*m->nlp, cfg);
  out[4] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  out[0] = r.iterations;
  out[1] = r.objective;
  out[2] = static_cast<double>(static_cast<int>(r.status));
  out[3] = r.restorations;
}

// ---------------------------------------------------------------- IPM vector ops
// Lifted bounds of the model's LiftedProblem: xl, xu [n], sl, su [m].
void gnr_lifted_bounds(void* h, double* xl, double* xu, double* sl, double* su) {
  auto& L = *static_cast<RefModel*>(h)->lifted;
  std::memcpy(xl, L.x_lower().data(), L.x_lower().size() * sizeof(double));
  std::memcpy(xu, L.x_upper().data(), L.x_upper().size() * sizeof(double));
  std::memcpy(sl, L.s_lower().data(), L.s_lower().size() * sizeof(double));
  std::memcpy(su, L.s_upper().data(), L.s_upper().size() * sizeof(double));
}

}  // extern "C"

namespace {
struct IpmView {
  size_t n, m;
  std::span<const double> xl, xu, sl, su;
};
IpmView view(void* h, const double* const* b) {
  auto& L = *static_cast<RefModel*>(h)->lifted;
  const size_t n = static_cast<size_t>(L.n()), m = static_cast<size_t>(L.m());
  return {n, m, {b[0], n}, {b[1], n}, {b[2], m}, {b[3], m}};
}
// arrays: x s y zlx zux zls zus (iterate) / the same order for residuals and directions
ipm::Iterate make_it(const IpmView& v, const double* const* a) {
  ipm::Iterate it;
  it.x.assign(a[0], a[0] + v.n);
  it.s.assign(a[1], a[1] + v.m);
  it.y.assign(a[2], a[2] + v.m);
  it.zlx.assign(a[3], a[3] + v.n);
  it.zux.assign(a[4], a[4] + v.n);
  it.zls.assign(a[5], a[5] + v.m);
  it.zus.assign(a[6], a[6] + v.m);
  return it;
}
ipm::Residuals make_res(const IpmView& v, const double* const* a) {
  ipm::Residuals r;
  r.px.assign(a[0], a[0] + v.n);
  r.ps.assign(a[1], a[1] + v.m);
  r.py.assign(a[2], a[2] + v.m);
  r.pzlx.assign(a[3], a[3] + v.n);
  r.pzux.assign(a[4], a[4] + v.n);
  r.pzls.assign(a[5], a[5] + v.m);
  r.pzus.assign(a[6], a[6] + v.m);
  return r;
}
ipm::Direction make_dir(const IpmView& v, const double* const* a) {
  ipm::Direction d;
  d.dx.assign(a[0], a[0] + v.n);
  d.ds.assign(a[1], a[1] + v.m);
  d.dy.assign(a[2], a[2] + v.m);
  d.dzlx.assign(a[3], a[3] + v.n);
  d.dzux.assign(a[4], a[4] + v.n);
  d.dzls.assign(a[5], a[5] + v.m);
  d.dzus.assign(a[6], a[6] + v.m);
  return d;
}
void put7(const std::vector<double>* v[7], double* const* out) {
  for (int k = 0; k < 7; ++k) std::memcpy(out[k], v[k]->data(), v[k]->size() * sizeof(double));
}
}  // namespace

extern "C" {

void gnr_ipm_jac_t(void* h, const double* jv, const double* y, double* out) {
  auto& L = *static_cast<RefModel*>(h)->lifted;
  const size_t nj = static_cast<size_t>(L.jac_nnz());
  ipm::jac_transpose_multiply(L.jac_rows(), L.jac_cols(), {jv, nj},
                              {y, static_cast<size_t>(L.m())}, {out, static_cast<size_t>(L.n())});
}

void gnr_ipm_jac(void* h, const double* jv, const double* x, double* out) {
  auto& L = *static_cast<RefModel*>(h)->lifted;
  const size_t nj = static_cast<size_t>(L.jac_nnz());
  ipm::jac_multiply(L.jac_rows(), L.jac_cols(), {jv, nj}, {x, static_cast<size_t>(L.n())},
                    {out, static_cast<size_t>(L.m())});
}

void gnr_ipm_residuals(void* h, const double* const* bounds, const double* const* it_a,
                       const double* grad, const double* g, const double* jv, double mu,
                       double* const* out) {
  auto& L = *static_cast<RefModel*>(h)->lifted;
  const IpmView v = view(h, bounds);
  const ipm::Iterate it = make_it(v, it_a);
  ipm::Residuals r;
  ipm::compute_residuals(it, {grad, v.n}, {g, v.m}, L.jac_rows(), L.jac_cols(),
                         {jv, static_cast<size_t>(L.jac_nnz())}, v.xl, v.xu, v.sl, v.su, mu, r);
  const std::vector<double>* o[7] = {&r.px, &r.ps, &r.py, &r.pzlx, &r.pzux, &r.pzls, &r.pzus};
  put7(o, out);
}

void gnr_ipm_condense(void* h, const double* const* bounds, const double* const* it_a,
                      const double* const* r_a, double* sx, double* ss, double* qx, double* qs) {
  const IpmView v = view(h, bounds);
  const ipm::Iterate it = make_it(v, it_a);
  const ipm::Residuals r = make_res(v, r_a);
  std::vector<double> a, b, c, d;
  ipm::bound_condensation(it, r, v.xl, v.xu, v.sl, v.su, a, b, c, d);
  std::memcpy(sx, a.data(), v.n * sizeof(double));
  std::memcpy(ss, b.data(), v.m * sizeof(double));
  std::memcpy(qx, c.data(), v.n * sizeof(double));
  std::memcpy(qs, d.data(), v.m * sizeof(double));
}

void gnr_ipm_ftb(void* h, const double* const* bounds, const double* const* it_a,
                 const double* const* d_a, double tau, double* out2) {
  const IpmView v = view(h, bounds);
  const ipm::StepSizes a = ipm::fraction_to_boundary(make_it(v, it_a), make_dir(v, d_a), v.xl,
                                                     v.xu, v.sl, v.su, tau);
  out2[0] = a.primal;
  out2[1] = a.dual;
}

double gnr_ipm_barrier(void* h, const double* const* bounds, double f, const double* x,
                       const double* sv, double mu) {
  const IpmView v = view(h, bounds);
  return ipm::barrier_value(f, {x, v.n}, {sv, v.m}, v.xl, v.xu, v.sl, v.su, mu);
}

double gnr_ipm_slope(void* h, const double* const* bounds, const double* grad,
                     const double* const* it_a, const double* const* d_a, double mu) {
  const IpmView v = view(h, bounds);
  return ipm::barrier_slope({grad, v.n}, make_it(v, it_a), make_dir(v, d_a), v.xl, v.xu, v.sl,
                            v.su, mu);
}

double gnr_ipm_violation(void* h, const double* g, const double* sv) {
  const size_t m = static_cast<size_t>(static_cast<RefModel*>(h)->lifted->m());
  return ipm::constraint_violation({g, m}, {sv, m});
}

void gnr_ipm_kkt_error(void* h, const double* const* bounds, const double* const* it_a,
                       const double* const* r_a, double mu, double* out3) {
  const IpmView v = view(h, bounds);
  const ipm::KktError e = ipm::kkt_error(make_it(v, it_a), make_res(v, r_a), mu, v.xl, v.xu,
                                         v.sl, v.su);
  out3[0] = e.stat;
  out3[1] = e.feas;
  out3[2] = e.comp;
}

// d_a: dx, ds in; dzlx dzux dzls dzus out (d_out[0..3])
void gnr_ipm_recover(void* h, const double* const* bounds, const double* const* it_a,
                     const double* const* r_a, const double* const* d_a, double* const* d_out) {
  const IpmView v = view(h, bounds);
  ipm::Direction d = make_dir(v, d_a);
  ipm::recover_bound_steps(make_it(v, it_a), make_res(v, r_a), v.xl, v.xu, v.sl, v.su, d);
  std::memcpy(d_out[0], d.dzlx.data(), v.n * sizeof(double));
  std::memcpy(d_out[1], d.dzux.data(), v.n * sizeof(double));
  std::memcpy(d_out[2], d.dzls.data(), v.m * sizeof(double));
  std::memcpy(d_out[3], d.dzus.data(), v.m * sizeof(double));
}

// The vector parts of CondensedKkt::solve (condensed.hpp:150-172) around the factor
// solve, on the model's reference KKT: its own A (jacobian_csr / jacobian_values) and
// its csr_matvec / csr_matvec_transpose.  The c / d / sd formulas are the ones
// assemble() stores (condensed.hpp:112-116).  rhs[n] before, ds/dy[m] from dx after.
void gnr_kkt_solve_parts(void* h, const double* qx, const double* qs, const double* qy,
                         const double* ss, double dw, double dc, const double* dx, double* rhs,
                         double* ds, double* dy) {
  auto* mdl = static_cast<RefModel*>(h);
  const auto& a = mdl->kkt->jacobian_csr();
  const auto av = mdl->kkt->jacobian_values();
  const size_t n = static_cast<size_t>(mdl->lifted->n()), m = static_cast<size_t>(a.nrows);
  std::vector<double> tm(m), c(m), sd(m);
  for (size_t i = 0; i < m; ++i) {
    sd[i] = ss[i] + dw;
    c[i] = 1.0 / (1.0 + dc * sd[i]);
    tm[i] = c[i] * qs[i] + (sd[i] * c[i]) * qy[i];
  }
  std::vector<double> r(n);
  sparse::csr_matvec_transpose(a, av, tm, r);
  for (size_t i = 0; i < n; ++i) rhs[i] = -(qx[i] + r[i]);
  sparse::csr_matvec(a, av, {dx, n}, tm);
  for (size_t i = 0; i < m; ++i) {
    ds[i] = c[i] * (tm[i] + qy[i] - dc * qs[i]);
    dy[i] = -qs[i] - sd[i] * ds[i];
  }
}

}  // extern "C"
