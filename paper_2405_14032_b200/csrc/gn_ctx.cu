// Context construction: layout, device SoA network tables, J/H COO structure
// and the lifted (fixed-variable) filter.
//
//   layout / row blocks / patterns   power/opf.hpp:16-60, 100-355
//   COO slot order (freeze)          model/pattern_model.hpp:158-207
//   lifted filter                    ipm/lifted.hpp:25-100
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <limits>

#include "gn_internal.cuh"

namespace gnb {

static int64_t g_launches = 0;
void count_launch(int n) { g_launches += n; }
int64_t launch_count() { return g_launches; }

// ---- per-kernel event timing (gn_profile_*)
struct ProfRec {
  std::string name;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  double ms = 0.0;
  int64_t launches = 0;
};
static std::atomic<bool> g_prof{false};
static std::vector<ProfRec> g_recs;
static std::mutex g_prof_mu;  // the registry is shared by every context / thread

KTimer::KTimer(const char* name, cudaStream_t stream) {
  if (!g_prof) return;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (size_t i = 0; i < g_recs.size(); ++i)
    if (g_recs[i].name == name) idx = static_cast<int>(i);
  if (idx < 0) {
    g_recs.push_back(ProfRec{name});
    idx = static_cast<int>(g_recs.size()) - 1;
  }
  s = stream;
  cudaEventCreate(&a);
  cudaEventRecord(a, s);
}
KTimer::~KTimer() {
  if (idx < 0) return;
  cudaEvent_t b;
  cudaEventCreate(&b);
  cudaEventRecord(b, s);
  std::lock_guard<std::mutex> lock(g_prof_mu);
  g_recs[idx].pending.push_back({a, b});
}

void profile_enable(bool on) { g_prof = on; }
bool profiling() { return g_prof; }
void profile_reset() {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (auto& r : g_recs)
    for (auto& e : r.pending) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  g_recs.clear();
}
int profile_count() {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (auto& r : g_recs) {
    for (auto& e : r.pending) {
      float ms = 0.f;
      cudaEventSynchronize(e.second);
      cudaEventElapsedTime(&ms, e.first, e.second);
      r.ms += ms;
      r.launches += 1;
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    r.pending.clear();
  }
  return static_cast<int>(g_recs.size());
}
const char* profile_get(int i, double* ms, int64_t* launches) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  if (i < 0 || i >= static_cast<int>(g_recs.size())) return nullptr;
  *ms = g_recs[i].ms;
  *launches = g_recs[i].launches;
  return g_recs[i].name.c_str();
}

OpfDims make_dims(int32_t T, int32_t N, int32_t L, int32_t G, int32_t D, int32_t LT,
                  int32_t GR, int32_t ref, int32_t t0, int32_t T_total) {
  OpfDims d{};
  d.T = T; d.N = N; d.L = L; d.G = G; d.D = D; d.LT = LT; d.GR = GR; d.ref = ref;
  d.t0 = t0;
  d.T_total = T_total < 0 ? T : T_total;
  d.prev = t0 > 0 ? 1 : 0;
  d.next = t0 + T < d.T_total ? 1 : 0;
  d.s_lo = d.prev ? 0 : 1;
  d.R = T - 1 + d.prev + d.next;
  const int64_t T64 = T;
  auto chk = [](int64_t v, const char* what) {
    if (v > std::numeric_limits<int32_t>::max())
      throw Error(GN_ERR_INVALID, std::string("problem too large for int32 indices: ") + what);
    return static_cast<int32_t>(v);
  };
  // variables (opf.hpp:135-183)
  d.pg0 = 0;
  d.qg0 = chk(G * T64, "n");
  d.p0 = chk(2 * G * T64, "n");
  d.q0 = chk(d.p0 + L * T64, "n");
  d.v0 = chk(d.q0 + L * T64, "n");
  d.th0 = chk(d.v0 + N * T64, "n");
  d.n_base = chk(d.th0 + N * T64, "n");
  d.gh_prev = d.n_base;
  d.gh_next = chk(d.gh_prev + (int64_t)(d.prev ? GR : 0), "n");
  d.n = chk(d.gh_next + (int64_t)(d.next ? GR : 0), "n");
  // rows (opf.hpp:186-230)
  d.bal_p0 = 0;
  d.bal_q0 = chk(N * T64, "m");
  d.flow_p0 = chk(2 * N * T64, "m");
  d.flow_q0 = chk(d.flow_p0 + L * T64, "m");
  d.therm0 = chk(d.flow_q0 + L * T64, "m");
  d.ang0 = chk(d.therm0 + LT * T64, "m");
  d.ramp0 = chk(d.ang0 + L * T64, "m");
  const int64_t ramp_rows = GR * std::max<int64_t>(d.R, 0);
  d.m = chk(d.ramp0 + ramp_rows, "m");
  // patterns: records and fields
  const int64_t nrec[K_COUNT] = {G * T64, 2 * L * T64, 2 * L * T64, G * T64, G * T64,
                                 D * T64, D * T64, L * T64, L * T64, LT * T64, L * T64,
                                 ramp_rows};
  const int k[K_COUNT] = {1, 1, 1, 1, 1, 0, 0, 5, 5, 2, 2, 2};
  const bool present[K_COUNT] = {true, true, true, true, true, true, true, true, true,
                                 LT > 0, true, ramp_rows > 0};
  int pid = 0;
  int64_t jo = 0, ho = 0;
  for (int q = 0; q < K_COUNT; ++q) {
    d.nrec[q] = present[q] ? nrec[q] : 0;
    if (!present[q]) {
      d.pid[q] = -1;
      d.jac_off[q] = -1;
      d.hess_off[q] = -1;
      continue;
    }
    d.pid[q] = pid++;
    if (q != K_COST) {
      d.jac_off[q] = jo;
      jo += nrec[q] * k[q];
    } else {
      d.jac_off[q] = -1;
    }
    d.hess_off[q] = ho;
    ho += nrec[q] * k[q] * (k[q] + 1) / 2;
  }
  d.nj = jo;
  d.nh = ho;
  chk(d.nj, "jac_nnz");
  chk(d.nh, "hess_nnz");
  return d;
}

// --------------------------------------------------------------- structure
// (a null jr / hr: that structure is not wanted by this call -- gn_jac_structure and
// gn_hess_structure each build only their own)
__device__ __forceinline__ void put_h(int32_t* hr, int32_t* hc, int64_t s, int32_t a,
                                      int32_t b) {
  if (!hr) return;
  hr[s] = a > b ? a : b;
  hc[s] = a < b ? a : b;
}
__device__ __forceinline__ void put_j(int32_t* jr, int32_t* jc, int64_t s, int32_t row,
                                      int32_t col) {
  if (!jr) return;
  jr[s] = row;
  jc[s] = col;
}

// Per (l,t): patterns 1, 2 (balance flows), 7, 8 (flow definitions), 10 (angle).
__global__ void k_struct_line(OpfDims d, DevNet net, int32_t* jr, int32_t* jc, int32_t* hr,
                              int32_t* hc) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (int64_t)d.L * d.T) return;
  const int32_t l = (int32_t)(r / d.T), t = (int32_t)(r - (int64_t)l * d.T);
  const int32_t f = net.lf[l], to = net.lt[l];
  const int32_t p = d.p0 + (int32_t)r, q = d.q0 + (int32_t)r;
  const int32_t vf = d.v0 + f * d.T + t, vt = d.v0 + to * d.T + t;
  const int32_t af = d.th0 + f * d.T + t, at = d.th0 + to * d.T + t;
  // balance flows: to-record (s=+1) then from-record (s=-1), opf.hpp:254-257
  int64_t s = d.jac_off[K_BAL_P_FLOW] + 2 * r;
  put_j(jr, jc, s, d.bal_p0 + to * d.T + t, p);
  put_j(jr, jc, s + 1, d.bal_p0 + f * d.T + t, p);
  s = d.jac_off[K_BAL_Q_FLOW] + 2 * r;
  put_j(jr, jc, s, d.bal_q0 + to * d.T + t, q);
  put_j(jr, jc, s + 1, d.bal_q0 + f * d.T + t, q);
  s = d.hess_off[K_BAL_P_FLOW] + 2 * r;
  put_h(hr, hc, s, p, p); put_h(hr, hc, s + 1, p, p);
  s = d.hess_off[K_BAL_Q_FLOW] + 2 * r;
  put_h(hr, hc, s, q, q); put_h(hr, hc, s + 1, q, q);
  // flow definitions, fields [flow, v_f, v_t, th_f, th_t]
  int32_t fp[5] = {p, vf, vt, af, at};
  int32_t fq[5] = {q, vf, vt, af, at};
  for (int kind = K_FLOW_P; kind <= K_FLOW_Q; ++kind) {
    const int32_t* fv = kind == K_FLOW_P ? fp : fq;
    const int32_t row = (kind == K_FLOW_P ? d.flow_p0 : d.flow_q0) + (int32_t)r;
    int64_t js = d.jac_off[kind] + 5 * r;
    for (int i = 0; i < 5; ++i) { put_j(jr, jc, js + i, row, fv[i]); }
    int64_t hs = d.hess_off[kind] + 15 * r;
    for (int j = 0; j < 5; ++j)
      for (int i = j; i < 5; ++i) put_h(hr, hc, hs++, fv[i], fv[j]);
  }
  // angle spread [th_f, th_t]
  s = d.jac_off[K_ANGLE] + 2 * r;
  put_j(jr, jc, s, d.ang0 + (int32_t)r, af);
  put_j(jr, jc, s + 1, d.ang0 + (int32_t)r, at);
  s = d.hess_off[K_ANGLE] + 3 * r;
  put_h(hr, hc, s, af, af); put_h(hr, hc, s + 1, at, af); put_h(hr, hc, s + 2, at, at);
}

// Per (g,t): patterns 0 (cost), 3, 4 (injections).
__global__ void k_struct_gen(OpfDims d, DevNet net, int32_t* jr, int32_t* jc, int32_t* hr,
                             int32_t* hc) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (int64_t)d.G * d.T) return;
  const int32_t g = (int32_t)(r / d.T), t = (int32_t)(r - (int64_t)g * d.T);
  const int32_t bus = net.gbus[g];
  const int32_t pg = d.pg0 + (int32_t)r, qg = d.qg0 + (int32_t)r;
  put_h(hr, hc, d.hess_off[K_COST] + r, pg, pg);
  int64_t s = d.jac_off[K_BAL_P_INJ] + r;
  put_j(jr, jc, s, d.bal_p0 + bus * d.T + t, pg);
  s = d.jac_off[K_BAL_Q_INJ] + r;
  put_j(jr, jc, s, d.bal_q0 + bus * d.T + t, qg);
  put_h(hr, hc, d.hess_off[K_BAL_P_INJ] + r, pg, pg);
  put_h(hr, hc, d.hess_off[K_BAL_Q_INJ] + r, qg, qg);
}

// Per (k,t) of rated lines: pattern 9 (thermal) [p, q].
__global__ void k_struct_thermal(OpfDims d, DevNet net, int32_t* jr, int32_t* jc,
                                 int32_t* hr, int32_t* hc) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (int64_t)d.LT * d.T) return;
  const int32_t k = (int32_t)(r / d.T), t = (int32_t)(r - (int64_t)k * d.T);
  const int32_t l = net.th_line[k];
  const int32_t p = d.p0 + l * d.T + t, q = d.q0 + l * d.T + t;
  const int64_t s = d.jac_off[K_THERMAL] + 2 * r;
  put_j(jr, jc, s, d.therm0 + (int32_t)r, p);
  put_j(jr, jc, s + 1, d.therm0 + (int32_t)r, q);
  const int64_t h = d.hess_off[K_THERMAL] + 3 * r;
  put_h(hr, hc, h, p, p); put_h(hr, hc, h + 1, q, p); put_h(hr, hc, h + 2, q, q);
}

// Per (k, t>=1) of ramping generators: pattern 11 [pg_t, pg_{t-1}].
__global__ void k_struct_ramp(OpfDims d, DevNet net, int32_t* jr, int32_t* jc, int32_t* hr,
                              int32_t* hc) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t Rk = d.R;
  if (Rk <= 0 || r >= (int64_t)d.GR * Rk) return;
  const int32_t k = (int32_t)(r / Rk), st = (int32_t)(r - (int64_t)k * Rk);
  const int32_t g = net.ramp_gen[k];
  const int32_t a = ramp_var(d, g, k, d.s_lo + st, true), b = ramp_var(d, g, k, d.s_lo + st, false);
  const int64_t s = d.jac_off[K_RAMP] + 2 * r;
  put_j(jr, jc, s, d.ramp0 + (int32_t)r, a);
  put_j(jr, jc, s + 1, d.ramp0 + (int32_t)r, b);
  const int64_t h = d.hess_off[K_RAMP] + 3 * r;
  put_h(hr, hc, h, a, a); put_h(hr, hc, h + 1, b, a); put_h(hr, hc, h + 2, b, b);
}

static unsigned blocks_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

void build_structure(gn_ctx* c, int32_t* jr, int32_t* jc, int32_t* hr, int32_t* hc) {
  const OpfDims& d = c->d;
  const DevNet net = c->net();
  const int bs = 256;
  if ((int64_t)d.L * d.T > 0) {
    k_struct_line<<<blocks_for((int64_t)d.L * d.T, bs), bs, 0, c->stream>>>(d, net, jr, jc, hr, hc);
    count_launch();
  }
  if ((int64_t)d.G * d.T > 0) {
    k_struct_gen<<<blocks_for((int64_t)d.G * d.T, bs), bs, 0, c->stream>>>(d, net, jr, jc, hr, hc);
    count_launch();
  }
  if (d.pid[K_THERMAL] >= 0) {
    k_struct_thermal<<<blocks_for((int64_t)d.LT * d.T, bs), bs, 0, c->stream>>>(d, net, jr, jc, hr, hc);
    count_launch();
  }
  if (d.pid[K_RAMP] >= 0) {
    k_struct_ramp<<<blocks_for((int64_t)d.GR * d.R, bs), bs, 0, c->stream>>>(d, net, jr, jc, hr, hc);
    count_launch();
  }
  GN_CK(cudaGetLastError());
}

// ------------------------------------------------------------------ lifted
// var i belongs to entity i / T in block order [pg G][qg G][p L][q L][v N][th N].
__global__ void k_free_flags(int32_t n, int32_t T, int32_t n_base, int32_t gh_next,
                             const uint8_t* fixed_ent, int32_t* flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i >= n_base) {  // ghost set-points: prev ghosts are fixed (halo values), next free
    flag[i] = i >= gh_next ? 1 : 0;
    return;
  }
  flag[i] = fixed_ent[i / T] ? 0 : 1;
}
__global__ void k_free_scatter(int32_t n, const int32_t* flag, const int32_t* pos,
                               int32_t* free_of_full, int32_t* full_of_free) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (flag[i]) {
    free_of_full[i] = pos[i];
    full_of_free[pos[i]] = (int32_t)i;
  } else {
    free_of_full[i] = -1;
  }
}
__global__ void k_pick_flags(int64_t nnz, const int32_t* rows, const int32_t* cols,
                             const int32_t* free_of_full, int both, int32_t* flag) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const bool keep = free_of_full[cols[k]] >= 0 && (!both || free_of_full[rows[k]] >= 0);
  flag[k] = keep ? 1 : 0;
}
__global__ void k_pick_scatter(int64_t nnz, const int32_t* rows, const int32_t* cols,
                               const int32_t* free_of_full, int map_rows, const int32_t* flag,
                               const int32_t* pos, int32_t* orow, int32_t* ocol,
                               int32_t* pick) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz || !flag[k]) return;
  const int32_t o = pos[k];
  orow[o] = map_rows ? free_of_full[rows[k]] : rows[k];
  ocol[o] = free_of_full[cols[k]];
  pick[o] = (int32_t)k;
}

// Exclusive prefix sum of int32 flags; returns the total.
int32_t exclusive_scan(const int32_t* flag, int32_t* pos, int64_t n, cudaStream_t s) {
  if (n == 0) return 0;
  size_t bytes = 0;
  GN_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag, pos, n, s));
  DBuf<unsigned char> tmp;
  tmp.alloc(bytes);
  GN_CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, flag, pos, n, s));
  count_launch();
  int32_t last_pos = 0, last_flag = 0;
  GN_CK(cudaMemcpyAsync(&last_pos, pos + n - 1, 4, cudaMemcpyDeviceToHost, s));
  GN_CK(cudaMemcpyAsync(&last_flag, flag + n - 1, 4, cudaMemcpyDeviceToHost, s));
  GN_CK(cudaStreamSynchronize(s));
  return last_pos + last_flag;
}

void build_lifted(gn_ctx* c) {
  const OpfDims& d = c->d;
  cudaStream_t s = c->stream;
  const int bs = 256;
  // fixed entities (xl == xu, lifted.hpp:140-147) from the per-entity boxes
  std::vector<uint8_t> fixed(static_cast<size_t>(2 * d.G + 2 * d.L + 2 * d.N) + 1, 0);
  size_t e = 0;
  for (int32_t g = 0; g < d.G; ++g) fixed[e++] = c->gen_pmin[g] == c->gen_pmax[g];
  for (int32_t g = 0; g < d.G; ++g) fixed[e++] = c->gen_qmin[g] == c->gen_qmax[g];
  e += 2 * static_cast<size_t>(d.L);  // flows are (-inf, inf)
  for (int32_t n = 0; n < d.N; ++n) fixed[e++] = c->bus_vmin[n] == c->bus_vmax[n];
  for (int32_t n = 0; n < d.N; ++n) fixed[e++] = (n == d.ref);  // th_ref box [0, 0]
  c->var_fixed.upload(fixed.data(), fixed.size(), s);
  c->fixed_ent.assign(fixed.begin(), fixed.begin() + (fixed.size() - 1));

  DBuf<int32_t> flag, pos;
  flag.alloc(static_cast<size_t>(d.n) + 1);
  pos.alloc(static_cast<size_t>(d.n) + 1);
  k_free_flags<<<blocks_for(d.n, bs), bs, 0, s>>>(d.n, d.T, d.n_base, d.gh_next, c->var_fixed.p,
                                                  flag.p);
  count_launch();
  c->n_free = exclusive_scan(flag.p, pos.p, d.n, s);
  c->free_of_full.alloc(static_cast<size_t>(d.n) + 1);
  c->full_of_free.alloc(static_cast<size_t>(c->n_free) + 1);
  k_free_scatter<<<blocks_for(d.n, bs), bs, 0, s>>>(d.n, flag.p, pos.p, c->free_of_full.p,
                                                   c->full_of_free.p);
  count_launch();

  // full structure, then order-preserving compaction (lifted.hpp:178-198)
  DBuf<int32_t> jr, jc, hr, hc;
  jr.alloc(d.nj + 1); jc.alloc(d.nj + 1); hr.alloc(d.nh + 1); hc.alloc(d.nh + 1);
  build_structure(c, jr.p, jc.p, hr.p, hc.p);

  flag.alloc(static_cast<size_t>(std::max(d.nj, d.nh)) + 1);
  pos.alloc(flag.n);
  k_pick_flags<<<blocks_for(d.nj, bs), bs, 0, s>>>(d.nj, jr.p, jc.p, c->free_of_full.p, 0, flag.p);
  count_launch();
  c->nj_l = exclusive_scan(flag.p, pos.p, d.nj, s);
  c->jr_l.alloc(c->nj_l + 1); c->jc_l.alloc(c->nj_l + 1); c->jpick.alloc(c->nj_l + 1);
  k_pick_scatter<<<blocks_for(d.nj, bs), bs, 0, s>>>(d.nj, jr.p, jc.p, c->free_of_full.p, 0,
                                                    flag.p, pos.p, c->jr_l.p, c->jc_l.p,
                                                    c->jpick.p);
  count_launch();
  k_pick_flags<<<blocks_for(d.nh, bs), bs, 0, s>>>(d.nh, hr.p, hc.p, c->free_of_full.p, 1, flag.p);
  count_launch();
  c->nh_l = exclusive_scan(flag.p, pos.p, d.nh, s);
  c->hr_l.alloc(c->nh_l + 1); c->hc_l.alloc(c->nh_l + 1); c->hpick.alloc(c->nh_l + 1);
  k_pick_scatter<<<blocks_for(d.nh, bs), bs, 0, s>>>(d.nh, hr.p, hc.p, c->free_of_full.p, 1,
                                                    flag.p, pos.p, c->hr_l.p, c->hc_l.p,
                                                    c->hpick.p);
  count_launch();
  GN_CK(cudaGetLastError());
  GN_CK(cudaStreamSynchronize(s));
  c->lifted = true;
}

// ------------------------------------------------------------------- bounds
// NlpProblem bounds on the host (opf.hpp:135-230).
void host_bounds(const gn_ctx* c, double* xl, double* xu, double* xs, double* rl,
                 double* ru) {
  const OpfDims& d = c->d;
  const double inf = std::numeric_limits<double>::infinity();
  const int64_t T = d.T;
  auto spread = [&](double* out, int32_t off, int32_t count, auto fn) {
    if (!out) return;
    for (int32_t e = 0; e < count; ++e) {
      const double v = fn(e);
      for (int64_t t = 0; t < T; ++t) out[off + e * T + t] = v;
    }
  };
  spread(xl, d.pg0, d.G, [&](int32_t g) { return c->gen_pmin[g]; });
  spread(xu, d.pg0, d.G, [&](int32_t g) { return c->gen_pmax[g]; });
  spread(xs, d.pg0, d.G, [&](int32_t g) { return c->gen_pstart[g]; });
  spread(xl, d.qg0, d.G, [&](int32_t g) { return c->gen_qmin[g]; });
  spread(xu, d.qg0, d.G, [&](int32_t g) { return c->gen_qmax[g]; });
  spread(xs, d.qg0, d.G, [&](int32_t g) { return c->gen_qstart[g]; });
  // flow starts from the stored voltage point (opf.hpp:148-158, network.hpp:76-82)
  std::vector<double> ps(d.L), qs(d.L);
  for (int32_t l = 0; l < d.L; ++l) {
    const int32_t f = c->line_from[l], to = c->line_to[l];
    const double vm = c->vm_start[f], vn = c->vm_start[to];
    const double dth = c->va_start[f] - c->va_start[to];
    const double co = std::cos(dth), si = std::sin(dth), g = c->line_g[l], b = c->line_b[l];
    ps[l] = g * vm * vm - vm * vn * (g * co + b * si);
    qs[l] = -b * vm * vm - vm * vn * (g * si - b * co);
  }
  spread(xl, d.p0, d.L, [&](int32_t) { return -inf; });
  spread(xu, d.p0, d.L, [&](int32_t) { return inf; });
  spread(xs, d.p0, d.L, [&](int32_t l) { return ps[l]; });
  spread(xl, d.q0, d.L, [&](int32_t) { return -inf; });
  spread(xu, d.q0, d.L, [&](int32_t) { return inf; });
  spread(xs, d.q0, d.L, [&](int32_t l) { return qs[l]; });
  spread(xl, d.v0, d.N, [&](int32_t n) { return c->bus_vmin[n]; });
  spread(xu, d.v0, d.N, [&](int32_t n) { return c->bus_vmax[n]; });
  spread(xs, d.v0, d.N, [&](int32_t n) { return c->vm_start[n]; });
  spread(xl, d.th0, d.N, [&](int32_t n) { return n == d.ref ? 0.0 : -inf; });
  spread(xu, d.th0, d.N, [&](int32_t n) { return n == d.ref ? 0.0 : inf; });
  spread(xs, d.th0, d.N, [&](int32_t n) { return n == d.ref ? 0.0 : c->va_start[n]; });
  // ghost set-points of a period shard: prev ghosts are fixed (their x entries
  // carry the halo values), next ghosts are free
  for (int32_t i = d.n_base; i < d.n; ++i) {
    const bool fixed = i < d.gh_next;
    if (xl) xl[i] = fixed ? 0.0 : -inf;
    if (xu) xu[i] = fixed ? 0.0 : inf;
    if (xs) xs[i] = 0.0;
  }
  if (rl || ru) {
    for (int32_t i = 0; i < d.therm0; ++i) {
      if (rl) rl[i] = 0.0;
      if (ru) ru[i] = 0.0;
    }
    for (int32_t k = 0; k < d.LT; ++k) {
      const double smax = c->line_smax[c->thermal_lines[k]];
      for (int64_t t = 0; t < T; ++t) {
        if (rl) rl[d.therm0 + k * T + t] = -inf;
        if (ru) ru[d.therm0 + k * T + t] = smax * smax;
      }
    }
    for (int32_t l = 0; l < d.L; ++l)
      for (int64_t t = 0; t < T; ++t) {
        if (rl) rl[d.ang0 + l * T + t] = c->line_amin[l];
        if (ru) ru[d.ang0 + l * T + t] = c->line_amax[l];
      }
    for (int32_t k = 0; k < d.GR; ++k) {
      const double r = c->gen_ramp[c->ramp_gens[k]];
      for (int64_t s = 0; s < d.R; ++s) {
        if (rl) rl[d.ramp0 + (int64_t)k * d.R + s] = -r;
        if (ru) ru[d.ramp0 + (int64_t)k * d.R + s] = r;
      }
    }
  }
}

}  // namespace gnb

gnb::DevNet gn_ctx::net() const {
  gnb::DevNet n{};
  n.lf = lf.p; n.lt = lt.p; n.lg = lg.p; n.lb = lb.p; n.l_therm = l_therm.p;
  n.th_line = th_line.p; n.gbus = gbus.p; n.c2 = c2.p; n.c1 = c1.p; n.c0 = c0.p;
  n.ramp_gen = ramp_gen.p; n.pd = pd.p; n.qd = qd.p;
  n.bl_ptr = bl_ptr.p; n.bl = bl.p; n.bg_ptr = bg_ptr.p; n.bg = bg.p;
  n.bd_ptr = bd_ptr.p; n.bd = bd.p; n.var_fixed = var_fixed.p;
  return n;
}
