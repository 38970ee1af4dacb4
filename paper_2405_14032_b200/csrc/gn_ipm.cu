// Device-resident interior-point vector operations.
//
// The reference IPM (ipm/solver.hpp) runs these on host vectors every
// iteration; with the callbacks and the KKT assembly on the device they are
// what keeps x, y, z and the residuals from crossing PCIe:
//
//   jac_transpose_multiply / jac_multiply   iterate.hpp:42-62
//   compute_residuals                       iterate.hpp:64-97
//   bound_condensation                      iterate.hpp:99-145
//   fraction_to_boundary                    iterate.hpp:147-198
//   barrier_value / barrier_slope           iterate.hpp:200-236
//   constraint_violation                    iterate.hpp:238-244
//   kkt_error                               iterate.hpp:246-298
//   recover_bound_steps                     condensed.hpp:187-212
//   CondensedKkt::solve, vector parts       condensed.hpp:150-172 (the LDL^T stays on the host)
//
// Element-wise results and the sparse products are bit-identical to the
// reference: every sum runs in the reference's order (COO order k for J^T y
// and J x, CSR row order for A^T v, per-row order for A v) and the library is
// built with -fmad=false.  Reductions over a whole vector (barrier value and
// slope, constraint violation, the kkt_error sums) use a fixed two-level tree:
// deterministic run to run, equal to the reference's sequential sums to
// rounding (1e-12 relative in the tests).  max/min reductions are exact.
#include <cub/cub.cuh>

#include "gn_eval.cuh"
#include "gn_ipm.cuh"


namespace gnb {

void compress_keys(uint64_t* keys, int64_t nnz, int32_t nrows, int32_t ncols, Csc& out,
                   cudaStream_t s);

namespace {

constexpr int kIB = 256;          // threads per block
// unroll of the grid-stride reduction loops (more loads in flight; the per-thread
// accumulation order is unchanged); tuning builds override it
#ifndef GN_RED_UNROLL
#define GN_RED_UNROLL 4
#endif
constexpr int kRedUnroll = GN_RED_UNROLL;
constexpr int kRedBlocks = 1184;  // 8 x 148 SMs: fixed grid of the reduction passes

unsigned nblk(int64_t n) { return (unsigned)((n + kIB - 1) / kIB); }

__device__ __forceinline__ bool has_lo(double b) { return b > -INFINITY; }
__device__ __forceinline__ bool has_hi(double b) { return b < INFINITY; }

__global__ void k_col_keys(int64_t n, const int32_t* __restrict__ c, uint64_t* key) {
  const int64_t i = (int64_t)blockIdx.x * kIB + threadIdx.x;
  if (i < n) key[i] = (uint64_t)(uint32_t)c[i];
}

__global__ void k_list_product(int32_t n, const int2* __restrict__ be,
                               const int32_t* __restrict__ src, const int32_t* __restrict__ oth,
                               const double* __restrict__ vals, const double* __restrict__ v,
                               double* __restrict__ out) {
  const int32_t c = blockIdx.x * kIB + threadIdx.x;
  if (c >= n) return;
  const int2 b = be[c];
  double acc = 0.0;
  for (int32_t q = b.x; q < b.y; ++q) acc += vals[src[q]] * v[oth[q]];
  out[c] = acc;
}

// list bounds and contributor "other" indices (see gn_ipm::jt_be)
__global__ void k_list_be(int32_t n, const int32_t* __restrict__ ptr,
                          const int32_t* __restrict__ seg, int2* __restrict__ be) {
  const int32_t c = blockIdx.x * kIB + threadIdx.x;
  if (c >= n) return;
  be[c] = ptr[c + 1] > ptr[c] ? make_int2(seg[ptr[c]], seg[ptr[c] + 1]) : make_int2(0, 0);
}
__global__ void k_list_oth(int64_t nnz, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ other, int32_t* __restrict__ oth) {
  const int64_t q = (int64_t)blockIdx.x * kIB + threadIdx.x;
  if (q < nnz) oth[q] = other[src[q]];
}

// ------------------------------------------------------------ residuals
// px = grad - J^T y - zlx + zux (J^T y in COO order), pzl/pzu with the bounds.
__global__ void k_res_x(int32_t n, const int2* __restrict__ be,
                        const int32_t* __restrict__ src, const double* __restrict__ jv,
                        const int32_t* __restrict__ oth, const double* __restrict__ y,
                        const double* __restrict__ grad, const double* __restrict__ x,
                        const double* __restrict__ zl, const double* __restrict__ zu,
                        const double* __restrict__ xl, const double* __restrict__ xu, double mu,
                        double* __restrict__ px, double* __restrict__ pzl,
                        double* __restrict__ pzu) {
  const int32_t i = blockIdx.x * kIB + threadIdx.x;
  if (i >= n) return;
  const int2 b = be[i];
  double jty = 0.0;
  for (int32_t q = b.x; q < b.y; ++q) jty += jv[src[q]] * y[oth[q]];
  px[i] = grad[i] - jty - zl[i] + zu[i];
  const double lo = xl[i], hi = xu[i], xi = x[i];
  pzl[i] = has_lo(lo) ? zl[i] * (xi - lo) - mu : 0.0;
  pzu[i] = has_hi(hi) ? zu[i] * (hi - xi) - mu : 0.0;
}

__global__ void k_res_s(int32_t m, const double* __restrict__ y, const double* __restrict__ g,
                        const double* __restrict__ s, const double* __restrict__ zl,
                        const double* __restrict__ zu, const double* __restrict__ sl,
                        const double* __restrict__ su, double mu, double* __restrict__ ps,
                        double* __restrict__ py, double* __restrict__ pzl,
                        double* __restrict__ pzu) {
  const int32_t i = blockIdx.x * kIB + threadIdx.x;
  if (i >= m) return;
  ps[i] = y[i] - zl[i] + zu[i];
  py[i] = g[i] - s[i];
  const double lo = sl[i], hi = su[i], si = s[i];
  pzl[i] = has_lo(lo) ? zl[i] * (si - lo) - mu : 0.0;
  pzu[i] = has_hi(hi) ? zu[i] * (hi - si) - mu : 0.0;
}

// --------------------------------------------------- bound condensation
__global__ void k_condense(int32_t n, const double* __restrict__ w, const double* __restrict__ zl,
                           const double* __restrict__ zu, const double* __restrict__ p,
                           const double* __restrict__ pzl, const double* __restrict__ pzu,
                           const double* __restrict__ lo_, const double* __restrict__ hi_,
                           double* __restrict__ sigma, double* __restrict__ q) {
  const int32_t i = blockIdx.x * kIB + threadIdx.x;
  if (i >= n) return;
  double sg = 0.0, qq = p[i];
  const double lo = lo_[i], hi = hi_[i];
  if (has_lo(lo)) {
    const double gap = w[i] - lo;
    sg += zl[i] / gap;
    qq += pzl[i] / gap;
  }
  if (has_hi(hi)) {
    const double gap = hi - w[i];
    sg += zu[i] / gap;
    qq -= pzu[i] / gap;
  }
  sigma[i] = sg;
  q[i] = qq;
}

// ---------------------------------------------------- recover bound steps
__global__ void k_recover(int32_t n, const double* __restrict__ w, const double* __restrict__ d,
                          const double* __restrict__ zl, const double* __restrict__ zu,
                          const double* __restrict__ pzl, const double* __restrict__ pzu,
                          const double* __restrict__ lo_, const double* __restrict__ hi_,
                          double* __restrict__ dzl, double* __restrict__ dzu) {
  const int32_t i = blockIdx.x * kIB + threadIdx.x;
  if (i >= n) return;
  const double lo = lo_[i], hi = hi_[i];
  dzl[i] = has_lo(lo) ? -(pzl[i] + zl[i] * d[i]) / (w[i] - lo) : 0.0;
  dzu[i] = has_hi(hi) ? (-pzu[i] + zu[i] * d[i]) / (hi - w[i]) : 0.0;
}

// ------------------------------------------------------------ reductions
// Block-level tree over kIB lanes (fixed shape); Op is sum, max or min.
enum RedOp { R_SUM = 0, R_MAX = 1, R_MIN = 2 };
template <int OP>
__device__ __forceinline__ double red_op(double a, double b) {
  if constexpr (OP == R_SUM) return a + b;
  else if constexpr (OP == R_MAX) return fmax(a, b);
  else return fmin(a, b);
}
template <int OP, int K>
__device__ __forceinline__ void block_reduce(double (&v)[K], double* out) {
  __shared__ double sm[K][kIB / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double a = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = red_op<OP>(a, __shfl_down_sync(0xffffffffu, a, o));
    if (lane == 0) sm[k][warp] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double a = sm[k][0];
      for (int w = 1; w < kIB / 32; ++w) a = red_op<OP>(a, sm[k][w]);
      out[k] = a;
    }
  }
  __syncthreads();
}

// kkt_error pass: sums (|z| present, count present, |y|) and maxima (|px|, |ps|, |py|, comp)
struct KktIn {
  int32_t n, m;
  const double *x, *s, *y, *zlx, *zux, *zls, *zus, *px, *ps, *py, *xl, *xu, *sl, *su;
  double mu;
};
__global__ void __launch_bounds__(kIB) k_kkt_err(KktIn a, double* __restrict__ part) {
  double sums[3] = {0.0, 0.0, 0.0}, maxs[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t total = (int64_t)a.n + a.m;
#pragma unroll kRedUnroll
  for (int64_t i = (int64_t)blockIdx.x * kIB + threadIdx.x; i < total; i += (int64_t)gridDim.x * kIB) {
    if (i < a.n) {
      const int32_t j = (int32_t)i;
      const double lo = a.xl[j], hi = a.xu[j];
      if (has_lo(lo)) {
        sums[0] += fabs(a.zlx[j]);
        sums[1] += 1.0;
        maxs[3] = fmax(maxs[3], fabs(a.zlx[j] * (a.x[j] - lo) - a.mu));
      }
      if (has_hi(hi)) {
        sums[0] += fabs(a.zux[j]);
        sums[1] += 1.0;
        maxs[3] = fmax(maxs[3], fabs(a.zux[j] * (hi - a.x[j]) - a.mu));
      }
      maxs[0] = fmax(maxs[0], fabs(a.px[j]));
    } else {
      const int32_t j = (int32_t)(i - a.n);
      const double lo = a.sl[j], hi = a.su[j];
      if (has_lo(lo)) {
        sums[0] += fabs(a.zls[j]);
        sums[1] += 1.0;
        maxs[3] = fmax(maxs[3], fabs(a.zls[j] * (a.s[j] - lo) - a.mu));
      }
      if (has_hi(hi)) {
        sums[0] += fabs(a.zus[j]);
        sums[1] += 1.0;
        maxs[3] = fmax(maxs[3], fabs(a.zus[j] * (hi - a.s[j]) - a.mu));
      }
      sums[2] += fabs(a.y[j]);
      maxs[1] = fmax(maxs[1], fabs(a.ps[j]));
      maxs[2] = fmax(maxs[2], fabs(a.py[j]));
    }
  }
  __shared__ double o[7];
  block_reduce<R_SUM, 3>(sums, o);
  block_reduce<R_MAX, 4>(maxs, o + 3);
  if (threadIdx.x == 0)
    for (int k = 0; k < 7; ++k) part[(int64_t)k * gridDim.x + blockIdx.x] = o[k];
}

__global__ void __launch_bounds__(kIB) k_kkt_err_final(const double* __restrict__ part, int nb,
                                                       int32_t m, double* __restrict__ out) {
  double sums[3] = {0.0, 0.0, 0.0}, maxs[4] = {0.0, 0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nb; b += kIB) {
    for (int k = 0; k < 3; ++k) sums[k] += part[(int64_t)k * nb + b];
    for (int k = 0; k < 4; ++k) maxs[k] = fmax(maxs[k], part[(int64_t)(3 + k) * nb + b]);
  }
  __shared__ double o[7];
  block_reduce<R_SUM, 3>(sums, o);
  block_reduce<R_MAX, 4>(maxs, o + 3);
  if (threadIdx.x == 0) {  // iterate.hpp:272-297
    const double z_sum = o[0], z_count = o[1], y_sum = o[2];
    const double s_max = 100.0;
    const double s_d = fmax(s_max, (y_sum + z_sum) / fmax(1.0, (double)m + z_count)) / s_max;
    const double s_c = fmax(s_max, z_sum / fmax(1.0, z_count)) / s_max;
    out[0] = fmax(o[3], o[4]) / s_d;  // stat
    out[1] = o[5];                    // feas
    out[2] = o[6] / s_c;              // comp
  }
}

// generic scalar reductions: barrier value / slope, constraint violation, fraction to boundary
enum ScalarKind { S_BARRIER = 0, S_SLOPE = 1, S_VIOL = 2, S_FTB = 3 };
struct ScalIn {
  int32_t n, m;
  const double *x, *s, *xl, *xu, *sl, *su, *grad, *dx, *ds, *g;
  const double *zlx, *zux, *zls, *zus, *dzlx, *dzux, *dzls, *dzus;
  double mu, tau;
};
template <int KIND>
__global__ void __launch_bounds__(kIB) k_scalar(ScalIn a, double* __restrict__ part) {
  double v[2] = {KIND == S_FTB ? 1.0 : 0.0, KIND == S_FTB ? 1.0 : 0.0};
  const int64_t total = (int64_t)a.n + a.m;
#pragma unroll kRedUnroll
  for (int64_t i = (int64_t)blockIdx.x * kIB + threadIdx.x; i < total; i += (int64_t)gridDim.x * kIB) {
    const bool isx = i < a.n;
    const int32_t j = isx ? (int32_t)i : (int32_t)(i - a.n);
    const double w = isx ? a.x[j] : a.s[j];
    const double lo = isx ? a.xl[j] : a.sl[j], hi = isx ? a.xu[j] : a.su[j];
    if constexpr (KIND == S_BARRIER) {  // sum of log gaps (iterate.hpp:201-218)
      if (has_lo(lo)) v[0] += log(w - lo);
      if (has_hi(hi)) v[0] += log(hi - w);
    } else if constexpr (KIND == S_SLOPE) {  // iterate.hpp:221-236
      const double d = isx ? a.dx[j] : a.ds[j];
      if (isx) v[0] += a.grad[j] * d;
      if (has_lo(lo)) v[0] -= a.mu * d / (w - lo);
      if (has_hi(hi)) v[0] += a.mu * d / (hi - w);
    } else if constexpr (KIND == S_VIOL) {  // iterate.hpp:239-244 (over m only)
      if (!isx) v[0] += fabs(a.g[j] - a.s[j]);
    } else {  // fraction to boundary (iterate.hpp:166-198): v[0] primal, v[1] dual
      const double d = isx ? a.dx[j] : a.ds[j];
      if (has_lo(lo) && d < 0.0) v[0] = fmin(v[0], -a.tau * (w - lo) / d);
      if (has_hi(hi) && d > 0.0) v[0] = fmin(v[0], a.tau * (hi - w) / d);
      const double zl = isx ? a.zlx[j] : a.zls[j], dzl = isx ? a.dzlx[j] : a.dzls[j];
      const double zu = isx ? a.zux[j] : a.zus[j], dzu = isx ? a.dzux[j] : a.dzus[j];
      if (has_lo(lo) && dzl < 0.0) v[1] = fmin(v[1], -a.tau * zl / dzl);
      if (has_hi(hi) && dzu < 0.0) v[1] = fmin(v[1], -a.tau * zu / dzu);
    }
  }
  __shared__ double o[2];
  block_reduce<KIND == S_FTB ? R_MIN : R_SUM, 2>(v, o);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = o[0];
    part[gridDim.x + blockIdx.x] = o[1];
  }
}

template <int KIND>
__global__ void __launch_bounds__(kIB) k_scalar_final(const double* __restrict__ part, int nb,
                                                      double f, double mu,
                                                      double* __restrict__ out) {
  double v[2] = {KIND == S_FTB ? 1.0 : 0.0, KIND == S_FTB ? 1.0 : 0.0};
  for (int b = threadIdx.x; b < nb; b += kIB) {
    if constexpr (KIND == S_FTB) {
      v[0] = fmin(v[0], part[b]);
      v[1] = fmin(v[1], part[nb + b]);
    } else {
      v[0] += part[b];
    }
  }
  __shared__ double o[2];
  block_reduce<KIND == S_FTB ? R_MIN : R_SUM, 2>(v, o);
  if (threadIdx.x == 0) {
    if constexpr (KIND == S_BARRIER) out[0] = f - mu * o[0];
    else if constexpr (KIND == S_FTB) {
      out[0] = o[0];
      out[1] = o[1];
    } else out[0] = o[0];
  }
}

// ------------------------------------------------ condensed solve (vector parts)
// tm = c*qs + d*qy with c = 1/(1 + dc*sd), d = sd*c, sd = sigma_s + dw (condensed.hpp:112-116, 152-154)
__global__ void k_solve_tm(int32_t m, const double* __restrict__ qs, const double* __restrict__ qy,
                           const double* __restrict__ ss, double dw, double dc,
                           double* __restrict__ tm) {
  const int32_t i = blockIdx.x * kIB + threadIdx.x;
  if (i >= m) return;
  const double sd = ss[i] + dw;
  const double c = 1.0 / (1.0 + dc * sd);
  const double d = sd * c;
  tm[i] = c * qs[i] + d * qy[i];
}
// rhs = -(qx + A^T tm): A^T tm per column in CSR row order (condensed.hpp:155-157)
__global__ void k_solve_rhs(int32_t n, const int2* __restrict__ be,
                            const int32_t* __restrict__ src, const double* __restrict__ av,
                            const int32_t* __restrict__ oth, const double* __restrict__ tm,
                            const double* __restrict__ qx, double* __restrict__ rhs) {
  const int32_t c = blockIdx.x * kIB + threadIdx.x;
  if (c >= n) return;
  const int2 b = be[c];
  double acc = 0.0;
  for (int32_t q = b.x; q < b.y; ++q) acc += av[src[q]] * tm[oth[q]];
  rhs[c] = -(qx[c] + acc);
}
// tm = A dx (per row, csr_matvec); ds = c*(tm + qy - dc*qs); dy = -qs - sd*ds (condensed.hpp:164-170)
__global__ void k_solve_finish(int32_t m, const int32_t* __restrict__ rowptr,
                               const int32_t* __restrict__ colidx, const double* __restrict__ av,
                               const double* __restrict__ dx, const double* __restrict__ qs,
                               const double* __restrict__ qy, const double* __restrict__ ss,
                               double dw, double dc, double* __restrict__ ds,
                               double* __restrict__ dy) {
  const int32_t r = blockIdx.x * kIB + threadIdx.x;
  if (r >= m) return;
  double acc = 0.0;
  for (int32_t k = rowptr[r]; k < rowptr[r + 1]; ++k) acc += av[k] * dx[colidx[k]];
  const double sd = ss[r] + dw;
  const double c = 1.0 / (1.0 + dc * sd);
  const double d_s = c * (acc + qy[r] - dc * qs[r]);
  ds[r] = d_s;
  dy[r] = -qs[r] - sd * d_s;
}

}  // namespace

// per-column / per-row contributor lists of a COO pattern (stable: ascending k)
static void build_lists(const int32_t* key32, int64_t nnz, int32_t nlists, Csc& out,
                        cudaStream_t s) {
  DBuf<uint64_t> key;
  key.alloc(static_cast<size_t>(nnz) + 1);
  if (nnz > 0) {
    k_col_keys<<<nblk(nnz), kIB, 0, s>>>(nnz, key32, key.p);
    count_launch();
  }
  compress_keys(key.p, nnz, 1, nlists, out, s);
}

}  // namespace gnb

// (definitions of the ABI functions are in gn_api.cu; these helpers do the work)
namespace gnb {

gn_ipm* ipm_create(gn_kkt* K, const double* xl, const double* xu, const double* sl,
                   const double* su, bool device_in) {
  if (!K->ctx || !K->ctx->lifted) throw Error(GN_ERR_INVALID, "ipm needs a lifted KKT");
  cudaStream_t s = K->stream;
  auto* P = new gn_ipm();
  P->device = K->device;
  P->K = K;
  P->n = K->n;
  P->m = K->m;
  P->nj = K->nj;
  const auto kind = device_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  auto put = [&](DBuf<double>& b, const double* src, int32_t cnt) {
    b.alloc(static_cast<size_t>(cnt) + 1);
    if (cnt) GN_CK(cudaMemcpyAsync(b.p, src, sizeof(double) * cnt, kind, s));
  };
  put(P->xl, xl, P->n);
  put(P->xu, xu, P->n);
  put(P->sl, sl, P->m);
  put(P->su, su, P->m);
  gn_ctx* c = K->ctx;
  build_lists(c->jc_l.p, K->nj, P->n, P->jt, s);
  build_lists(c->jr_l.p, K->nj, P->m, P->jr, s);
  build_lists(K->A.idx.p, K->annz, P->n, P->at, s);  // CSR positions are row-major: stable by column
  auto flatten = [&](const Csc& L, int32_t nl, const int32_t* other, int64_t nnz, DBuf<int2>& be,
                     DBuf<int32_t>& oth) {
    be.alloc(static_cast<size_t>(nl) + 1);
    oth.alloc(static_cast<size_t>(nnz) + 1);
    if (nl > 0) {
      k_list_be<<<nblk(nl), kIB, 0, s>>>(nl, L.ptr.p, L.seg.p, be.p);
      count_launch();
    }
    if (nnz > 0) {
      k_list_oth<<<(unsigned)((nnz + kIB - 1) / kIB), kIB, 0, s>>>(nnz, L.src.p, other, oth.p);
      count_launch();
    }
  };
  flatten(P->jt, P->n, c->jr_l.p, K->nj, P->jt_be, P->jt_oth);
  flatten(P->jr, P->m, c->jc_l.p, K->nj, P->jr_be, P->jr_oth);
  flatten(P->at, P->n, K->arow.p, K->annz, P->at_be, P->at_oth);
  P->part.alloc(static_cast<size_t>(kRedBlocks) * 8);
  P->scratch.alloc(static_cast<size_t>(P->m) + 1);
  GN_CK(cudaStreamSynchronize(s));
  return P;
}

void ipm_jac_t(gn_ipm* P, const double* jv, const double* y, double* out, cudaStream_t s) {
  {
    KTimer kt("k_ipm_jac_t", s);
    k_list_product<<<nblk(P->n), kIB, 0, s>>>(P->n, P->jt_be.p, P->jt.src.p, P->jt_oth.p, jv, y,
                                              out);
  }
  count_launch();
}
void ipm_jac(gn_ipm* P, const double* jv, const double* x, double* out, cudaStream_t s) {
  {
    KTimer kt("k_ipm_jac", s);
    k_list_product<<<nblk(P->m), kIB, 0, s>>>(P->m, P->jr_be.p, P->jr.src.p, P->jr_oth.p, jv, x,
                                              out);
  }
  count_launch();
}

void ipm_residuals(gn_ipm* P, const gn_iterate& it, const double* grad, const double* g,
                   const double* jv, double mu, const gn_residuals& r, cudaStream_t s) {
  {
    KTimer kt("k_ipm_res_x", s);
    k_res_x<<<nblk(P->n), kIB, 0, s>>>(P->n, P->jt_be.p, P->jt.src.p, jv, P->jt_oth.p, it.y,
                                       grad, it.x, it.zlx, it.zux, P->xl.p, P->xu.p, mu, r.px,
                                       r.pzlx, r.pzux);
  }
  count_launch();
  {
    KTimer kt("k_ipm_res_s", s);
    k_res_s<<<nblk(P->m), kIB, 0, s>>>(P->m, it.y, g, it.s, it.zls, it.zus, P->sl.p, P->su.p,
                                       mu, r.ps, r.py, r.pzls, r.pzus);
  }
  count_launch();
}

void ipm_condense(gn_ipm* P, const gn_iterate& it, const gn_residuals& r, double* sx, double* ss,
                  double* qx, double* qs, cudaStream_t s) {
  {
    KTimer kt("k_ipm_condense_x", s);
    k_condense<<<nblk(P->n), kIB, 0, s>>>(P->n, it.x, it.zlx, it.zux, r.px, r.pzlx, r.pzux, P->xl.p,
                                          P->xu.p, sx, qx);
  }
  count_launch();
  {
    KTimer kt("k_ipm_condense_s", s);
    k_condense<<<nblk(P->m), kIB, 0, s>>>(P->m, it.s, it.zls, it.zus, r.ps, r.pzls, r.pzus, P->sl.p,
                                          P->su.p, ss, qs);
  }
  count_launch();
}

void ipm_recover(gn_ipm* P, const gn_iterate& it, const gn_residuals& r, const gn_direction& d,
                 cudaStream_t s) {
  {
    KTimer kt("k_ipm_recover_x", s);
    k_recover<<<nblk(P->n), kIB, 0, s>>>(P->n, it.x, d.dx, it.zlx, it.zux, r.pzlx, r.pzux, P->xl.p,
                                         P->xu.p, d.dzlx, d.dzux);
  }
  count_launch();
  {
    KTimer kt("k_ipm_recover_s", s);
    k_recover<<<nblk(P->m), kIB, 0, s>>>(P->m, it.s, d.ds, it.zls, it.zus, r.pzls, r.pzus, P->sl.p,
                                         P->su.p, d.dzls, d.dzus);
  }
  count_launch();
}

void ipm_kkt_error(gn_ipm* P, const gn_iterate& it, const gn_residuals& r, double mu, double* out,
                   cudaStream_t s) {
  KktIn a{P->n, P->m, it.x, it.s, it.y, it.zlx, it.zux, it.zls, it.zus, r.px, r.ps, r.py,
          P->xl.p, P->xu.p, P->sl.p, P->su.p, mu};
  {
    KTimer kt("k_ipm_kkt_err", s);
    k_kkt_err<<<kRedBlocks, kIB, 0, s>>>(a, P->part.p);
  }
  count_launch();
  {
    KTimer kt("k_ipm_kkt_err_final", s);
    k_kkt_err_final<<<1, kIB, 0, s>>>(P->part.p, kRedBlocks, P->m, out);
  }
  count_launch();
}

static ScalIn scal(gn_ipm* P) {
  ScalIn a{};
  a.n = P->n;
  a.m = P->m;
  a.xl = P->xl.p; a.xu = P->xu.p; a.sl = P->sl.p; a.su = P->su.p;
  return a;
}

void ipm_barrier(gn_ipm* P, double f, const double* x, const double* sv, double mu, double* out,
                 cudaStream_t s) {
  ScalIn a = scal(P);
  a.x = x; a.s = sv; a.mu = mu;
  {
    KTimer kt("k_ipm_barrier", s);
    k_scalar<S_BARRIER><<<kRedBlocks, kIB, 0, s>>>(a, P->part.p);
  }
  count_launch();
  {
    KTimer kt("k_ipm_final", s);
    k_scalar_final<S_BARRIER><<<1, kIB, 0, s>>>(P->part.p, kRedBlocks, f, mu, out);
  }
  count_launch();
}

void ipm_slope(gn_ipm* P, const double* grad, const gn_iterate& it, const gn_direction& d,
               double mu, double* out, cudaStream_t s) {
  ScalIn a = scal(P);
  a.x = it.x; a.s = it.s; a.grad = grad; a.dx = d.dx; a.ds = d.ds; a.mu = mu;
  {
    KTimer kt("k_ipm_slope", s);
    k_scalar<S_SLOPE><<<kRedBlocks, kIB, 0, s>>>(a, P->part.p);
  }
  count_launch();
  {
    KTimer kt("k_ipm_final", s);
    k_scalar_final<S_SLOPE><<<1, kIB, 0, s>>>(P->part.p, kRedBlocks, 0.0, mu, out);
  }
  count_launch();
}

void ipm_violation(gn_ipm* P, const double* g, const double* sv, double* out, cudaStream_t s) {
  ScalIn a = scal(P);
  a.g = g; a.s = sv; a.x = sv;  // x is not read for the m-range
  a.n = 0;                      // m entries only
  {
    KTimer kt("k_ipm_violation", s);
    k_scalar<S_VIOL><<<kRedBlocks, kIB, 0, s>>>(a, P->part.p);
  }
  count_launch();
  {
    KTimer kt("k_ipm_final", s);
    k_scalar_final<S_VIOL><<<1, kIB, 0, s>>>(P->part.p, kRedBlocks, 0.0, 0.0, out);
  }
  count_launch();
}

void ipm_ftb(gn_ipm* P, const gn_iterate& it, const gn_direction& d, double tau, double* out,
             cudaStream_t s) {
  ScalIn a = scal(P);
  a.x = it.x; a.s = it.s; a.dx = d.dx; a.ds = d.ds;
  a.zlx = it.zlx; a.zux = it.zux; a.zls = it.zls; a.zus = it.zus;
  a.dzlx = d.dzlx; a.dzux = d.dzux; a.dzls = d.dzls; a.dzus = d.dzus;
  a.tau = tau;
  {
    KTimer kt("k_ipm_ftb", s);
    k_scalar<S_FTB><<<kRedBlocks, kIB, 0, s>>>(a, P->part.p);
  }
  count_launch();
  {
    KTimer kt("k_ipm_final", s);
    k_scalar_final<S_FTB><<<1, kIB, 0, s>>>(P->part.p, kRedBlocks, 0.0, 0.0, out);
  }
  count_launch();
}

void kkt_solve_rhs(gn_ipm* P, const double* qx, const double* qs, const double* qy,
                   const double* ss, double dw, double dc, double* rhs, double* tm,
                   cudaStream_t s) {
  gn_kkt* K = P->K;
  {
    KTimer kt("k_ipm_solve_tm", s);
    k_solve_tm<<<nblk(P->m), kIB, 0, s>>>(P->m, qs, qy, ss, dw, dc, tm);
  }
  count_launch();
  {
    KTimer kt("k_ipm_solve_rhs", s);
    k_solve_rhs<<<nblk(P->n), kIB, 0, s>>>(P->n, P->at_be.p, P->at.src.p, K->avals.p, P->at_oth.p,
                                           tm, qx, rhs);
  }
  count_launch();
}

void kkt_solve_finish(gn_ipm* P, const double* dx, const double* qs, const double* qy,
                      const double* ss, double dw, double dc, double* ds, double* dy,
                      cudaStream_t s) {
  gn_kkt* K = P->K;
  {
    KTimer kt("k_ipm_solve_finish", s);
    k_solve_finish<<<nblk(P->m), kIB, 0, s>>>(P->m, K->A.ptr.p, K->A.idx.p, K->avals.p, dx, qs, qy,
                                              ss, dw, dc, ds, dy);
  }
  count_launch();
}

}  // namespace gnb
