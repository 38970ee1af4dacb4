// Internal declarations shared by the CUDA translation units of libgridnlp_b200.
// Nothing here crosses the C-ABI (include/gridnlp_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gridnlp_b200.h"

namespace gnb {

// Host-side error carrying a C-ABI status code (GN_ERR_*).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GN_CK(expr)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw ::gnb::Error(GN_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

void count_launch(int n = 1);

// Host <-> device copies of the host-memory modes (gn_hostio.cu): pinned bounce buffers and
// parallel host copies for pageable caller memory; both return when the copy is complete.
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);

// Optional per-kernel CUDA-event timing (gn_profile_*): RAII around a launch.
struct KTimer {
  int idx = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t a = nullptr;
  KTimer(const char* name, cudaStream_t stream);
  ~KTimer();
};

// Owning device buffer (cudaMalloc / cudaFree on the current device).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    n = count;
    if (count) GN_CK(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) h2d(p, h, count * sizeof(T), s);
  }
  std::vector<T> download(cudaStream_t s) const {
    std::vector<T> h(n);
    if (n) {
      GN_CK(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
      GN_CK(cudaStreamSynchronize(s));
    }
    return h;
  }
};

// Pattern kinds in the reference's registration order (opf.hpp:236-351).  The
// registration *id* of thermal/angle/ramp depends on which optional patterns
// exist (thermal only if LT>0, ramp only if GR*(T-1)>0); OpfDims::pid maps.
enum Kind {
  K_COST = 0, K_BAL_P_FLOW, K_BAL_Q_FLOW, K_BAL_P_INJ, K_BAL_Q_INJ, K_BAL_P_LOAD,
  K_BAL_Q_LOAD, K_FLOW_P, K_FLOW_Q, K_THERMAL, K_ANGLE, K_RAMP, K_COUNT
};

// Closed-form layout (OpfLayout, opf.hpp:16-60) and COO offsets (freeze,
// pattern_model.hpp:158-207).
struct OpfDims {
  int32_t T, N, L, G, D, LT, GR, ref;
  // period shard [t0, t0 + T) of a T_total-period horizon; a full
  // problem is t0 = 0, T_total = T.  Ramp steps s = s_lo .. s_hi (R per ramp
  // generator) may reference ghost set-points pg(-1) (prev, fixed, halo from
  // rank r-1) and pg(T) (next, free; its rows are owned by rank r+1), stored
  // after the regular blocks: [n_base, gh_prev + GR) and [gh_next, gh_next + GR).
  int32_t t0, T_total, prev, next, s_lo, R, n_base, gh_prev, gh_next;
  int32_t pg0, qg0, p0, q0, v0, th0, n;
  int32_t bal_p0, bal_q0, flow_p0, flow_q0, therm0, ang0, ramp0, m;
  int64_t jac_off[K_COUNT], hess_off[K_COUNT], nrec[K_COUNT];
  int32_t pid[K_COUNT];  // registration id or -1 when the pattern is absent
  int64_t nj, nh;
};

OpfDims make_dims(int32_t T, int32_t N, int32_t L, int32_t G, int32_t D, int32_t LT,
                  int32_t GR, int32_t ref, int32_t t0 = 0, int32_t T_total = -1);

// variable of ramp step s (s = 0..T): pg(s) (a = true) or pg(s-1) (a = false)
#ifdef __CUDACC__
__host__ __device__
#endif
inline int32_t ramp_var(const OpfDims& d, int32_t g, int32_t k, int32_t s, bool a) {
  const int32_t p = a ? s : s - 1;
  if (p < 0) return d.gh_prev + k;
  if (p >= d.T) return d.gh_next + k;
  return d.pg0 + g * d.T + p;
}

// Device pointers to the SoA network tables consumed by the kernels.
struct DevNet {
  const int32_t *lf, *lt;      // [L]
  const double *lg, *lb;       // [L]
  const int32_t* l_therm;      // [L] thermal slot k or -1
  const int32_t* th_line;      // [LT] line of thermal slot
  const int32_t* gbus;         // [G]
  const double *c2, *c1, *c0;  // [G]
  const int32_t* ramp_gen;     // [GR]
  const double *pd, *qd;       // [D*T] entity-major (j*T + t)
  const int32_t *bl_ptr, *bl;  // bus -> (l<<1 | is_from), ascending l
  const int32_t *bg_ptr, *bg;  // bus -> generators, ascending
  const int32_t *bd_ptr, *bd;  // bus -> loads, ascending
  const uint8_t* var_fixed;    // per (block, entity): 6 blocks laid out like x / T
};

// Drop one dependent's reference on a context (frees it when destroyed and unreferenced).
void ctx_unref(gn_ctx* c);

// Status word: lexicographic min of (pattern id << 32 | record) over failures.
constexpr unsigned long long kNoFail = ~0ull;

}  // namespace gnb

// The context object behind the opaque C handle.
struct gn_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t owned_stream = nullptr;  // created here; destroyed with the object
  int refs = 0;         // live objects built on this one (KKTs / IPMs)
  bool closed = false;  // destroy requested; freed when refs drops to 0
  gnb::OpfDims d{};
  // host copies of the network (bounds, starts)
  std::vector<double> bus_vmin, bus_vmax, vm_start, va_start;
  std::vector<int32_t> line_from, line_to;
  std::vector<double> line_g, line_b, line_smax, line_amin, line_amax;
  std::vector<int32_t> gen_bus;
  std::vector<double> gen_pmin, gen_pmax, gen_qmin, gen_qmax, gen_ramp, gen_c2, gen_c1,
      gen_c0, gen_pstart, gen_qstart;
  std::vector<int32_t> thermal_lines, ramp_gens;
  // device tables
  gnb::DBuf<int32_t> lf, lt, l_therm, th_line, gbus, ramp_gen, bl_ptr, bl, bg_ptr, bg, bd_ptr, bd;
  gnb::DBuf<double> lg, lb, c2, c1, c0, pd, qd;
  gnb::DBuf<uint8_t> var_fixed;  // per-entity fixed flags (block order), see DevNet
  std::vector<uint8_t> fixed_ent;  // host copy
  gnb::DBuf<unsigned long long> status;
  gnb::DBuf<double> fpart;       // objective partial sums
  // host-mode staging
  gnb::DBuf<double> sx, sw, sout;
  // lifted problem
  bool lifted = false;
  double relax = 0.0;
  int32_t n_free = 0;
  int64_t nj_l = 0, nh_l = 0;
  gnb::DBuf<int32_t> free_of_full, full_of_free, jr_l, jc_l, jpick, hr_l, hc_l, hpick;
  // lifted evaluations (gn_lifted_eval_*): the full-space point with the fixed entries at
  // their pinned values (filled once), the free-variable upload and the lifted output
  gnb::DBuf<double> lx, lxin, lout;
  bool lx_ready = false;
  gnb::DevNet net() const;
};
