// Condensed-KKT structure and assembly on the device.
//
//   compress_to_csc / compress_to_csr  sparse/matrix.hpp:45-97  (GPU radix sort on
//                                      64-bit (col,row) keys; stable, so each
//                                      compressed slot's contributors stay in
//                                      ascending COO order)
//   CondensedKkt ctor                  ipm/condensed.hpp:29-90
//   set_jacobian (scatter_values)      ipm/condensed.hpp:99-101, matrix.hpp:100-106
//   assemble                           ipm/condensed.hpp:105-135
//
// Determinism: no atomics.  Every compressed slot is produced by one thread that
// sums its contributor list in the reference's order (0 (+) H in COO order (+)
// AtDA pairs in (r, ka, kb) order (+) dw + sigma_x), so with the same inputs
// the values are bit-identical to the reference's sequential scatter.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gn_kkt.cuh"

namespace gnb {

static unsigned nblk(int64_t n, int bs = 256) { return (unsigned)((n + bs - 1) / bs); }

static int bit_length(uint64_t v) {
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

__global__ void k_iota(int64_t n, int32_t* v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}
__global__ void k_run_flags(int64_t n, const uint64_t* key, int32_t* flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}
__global__ void k_run_emit(int64_t n, const uint64_t* key, const int32_t* flag,
                           const int32_t* pos, const int32_t* src, uint64_t nrows,
                           int32_t* idx, int32_t* ucol, int32_t* seg, int32_t* slot) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t s = pos[i] + flag[i] - 1;  // inclusive position - 1
  if (flag[i]) {
    idx[s] = (int32_t)(key[i] % nrows);
    ucol[s] = (int32_t)(key[i] / nrows);
    seg[s] = (int32_t)i;
  }
  slot[src[i]] = s;
}
__global__ void k_colptr(int32_t ncols, int32_t nnz, const int32_t* ucol, int32_t* ptr) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c > ncols) return;
  int32_t lo = 0, hi = nnz;  // first position with ucol >= c
  while (lo < hi) {
    const int32_t mid = lo + (hi - lo) / 2;
    if (ucol[mid] < c) lo = mid + 1; else hi = mid;
  }
  ptr[c] = lo;
}

void compress_keys(uint64_t* keys, int64_t nnz, int32_t nrows, int32_t ncols, Csc& out,
                   cudaStream_t s) {
  if (nnz > 0x7fffffffLL) throw Error(GN_ERR_INVALID, "compress: more than 2^31-1 entries");
  out.ptr.alloc(static_cast<size_t>(ncols) + 1);
  out.slot.alloc(static_cast<size_t>(nnz) + 1);
  if (nnz == 0) {
    GN_CK(cudaMemsetAsync(out.ptr.p, 0, sizeof(int32_t) * (ncols + 1), s));
    out.idx.alloc(1); out.seg.alloc(1); out.src.alloc(1);
    GN_CK(cudaMemsetAsync(out.seg.p, 0, sizeof(int32_t), s));
    out.nnz = 0;
    return;
  }
  DBuf<int32_t> vin;
  DBuf<uint64_t> kout;
  vin.alloc(nnz);
  kout.alloc(nnz);
  out.src.alloc(nnz);
  k_iota<<<nblk(nnz), 256, 0, s>>>(nnz, vin.p);
  count_launch();
  const int end_bit = std::max(1, bit_length((uint64_t)nrows * (uint64_t)ncols));
  size_t bytes = 0;
  GN_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, kout.p, vin.p, out.src.p, nnz,
                                        0, end_bit, s));
  {
    DBuf<unsigned char> tmp;
    tmp.alloc(bytes);
    GN_CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys, kout.p, vin.p, out.src.p, nnz,
                                          0, end_bit, s));
    count_launch();
    GN_CK(cudaStreamSynchronize(s));
  }
  vin.release();
  DBuf<int32_t> flag, pos, ucol;
  flag.alloc(nnz);
  pos.alloc(nnz);
  k_run_flags<<<nblk(nnz), 256, 0, s>>>(nnz, kout.p, flag.p);
  count_launch();
  out.nnz = exclusive_scan(flag.p, pos.p, nnz, s);
  out.idx.alloc(static_cast<size_t>(out.nnz) + 1);
  out.seg.alloc(static_cast<size_t>(out.nnz) + 1);
  ucol.alloc(static_cast<size_t>(out.nnz) + 1);
  k_run_emit<<<nblk(nnz), 256, 0, s>>>(nnz, kout.p, flag.p, pos.p, out.src.p, (uint64_t)nrows,
                                       out.idx.p, ucol.p, out.seg.p, out.slot.p);
  count_launch();
  const int32_t tail = (int32_t)nnz;
  GN_CK(cudaMemcpyAsync(out.seg.p + out.nnz, &tail, 4, cudaMemcpyHostToDevice, s));
  k_colptr<<<nblk((int64_t)ncols + 1), 256, 0, s>>>(ncols, out.nnz, ucol.p, out.ptr.p);
  count_launch();
  GN_CK(cudaGetLastError());
  GN_CK(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------- KKT build
__global__ void k_range_check(int64_t nnz, const int32_t* r, const int32_t* c, int32_t nr,
                              int32_t nc, int32_t* bad) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  if (r[k] < 0 || r[k] >= nr || c[k] < 0 || c[k] >= nc) atomicOr(bad, 1);
}
// A as CSR = CSC of the transpose: key = row * n + col.
__global__ void k_keys_jac(int64_t nnz, const int32_t* jr, const int32_t* jc, uint64_t n,
                           uint64_t* key) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) key[k] = (uint64_t)jr[k] * n + (uint64_t)jc[k];
}
// Hessian entries as (max, min): CSC key = col * n + row (condensed.hpp:47-53).
__global__ void k_keys_hess(int64_t nnz, const int32_t* hr, const int32_t* hc, uint64_t n,
                            uint64_t* key) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int32_t a = hr[k], b = hc[k];
  const uint64_t row = a > b ? a : b, col = a < b ? a : b;
  key[k] = col * n + row;
}
__global__ void k_pair_count(int32_t m, const int32_t* rowptr, int64_t* cnt) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const int64_t len = rowptr[r + 1] - rowptr[r];
  cnt[r] = len * (len + 1) / 2;
}
// Row pairs (colidx[ka], colidx[kb]), kb <= ka, in (r, ka, kb) order (condensed.hpp:62-70).
__global__ void k_pairs(int32_t m, const int32_t* rowptr, const int32_t* colidx,
                        const int64_t* poff, uint64_t n, uint64_t* key, int32_t* pka,
                        int32_t* pkb, int32_t* arow) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  int64_t p = poff[r];
  const int32_t a0 = rowptr[r], a1 = rowptr[r + 1];
  for (int32_t ka = a0; ka < a1; ++ka) {
    arow[ka] = (int32_t)r;
    for (int32_t kb = a0; kb <= ka; ++kb, ++p) {
      key[p] = (uint64_t)colidx[kb] * n + (uint64_t)colidx[ka];
      pka[p] = ka;
      pkb[p] = kb;
    }
  }
}
__global__ void k_keys_diag(int32_t n, uint64_t* key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = (uint64_t)i * (uint64_t)n + (uint64_t)i;
}

void kkt_build(gn_kkt* K, const int32_t* jr, const int32_t* jc, const int32_t* hr,
               const int32_t* hc) {
  cudaStream_t s = K->stream;
  const int32_t n = K->n, m = K->m;
  {
    DBuf<int32_t> bad;
    bad.alloc(1);
    GN_CK(cudaMemsetAsync(bad.p, 0, 4, s));
    if (K->nj) { k_range_check<<<nblk(K->nj), 256, 0, s>>>(K->nj, jr, jc, m, n, bad.p); count_launch(); }
    if (K->nh) { k_range_check<<<nblk(K->nh), 256, 0, s>>>(K->nh, hr, hc, n, n, bad.p); count_launch(); }
    int32_t hb = 0;
    GN_CK(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
    GN_CK(cudaStreamSynchronize(s));
    if (hb) throw Error(GN_ERR_INVALID, "compress_to_csc: coordinate out of range");
  }
  // ---- CSR(A) and jac_slots
  {
    DBuf<uint64_t> key;
    key.alloc(K->nj + 1);
    if (K->nj) { k_keys_jac<<<nblk(K->nj), 256, 0, s>>>(K->nj, jr, jc, (uint64_t)n, key.p); count_launch(); }
    compress_keys(key.p, K->nj, n, m, K->A, s);
  }
  K->annz = K->A.nnz;
  K->avals.alloc(static_cast<size_t>(K->annz) + kGuard);  // tail guard: gn_debug_kkt_guard
  GN_CK(cudaMemsetAsync(K->avals.p, 0, sizeof(double) * (K->annz + kGuard), s));
  // ---- pair offsets
  DBuf<int64_t> cnt, poff;
  cnt.alloc(static_cast<size_t>(m) + 1);
  poff.alloc(static_cast<size_t>(m) + 1);
  if (m) { k_pair_count<<<nblk(m), 256, 0, s>>>(m, K->A.ptr.p, cnt.p); count_launch(); }
  GN_CK(cudaMemsetAsync(cnt.p + m, 0, sizeof(int64_t), s));
  {
    size_t bytes = 0;
    GN_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, poff.p, (int64_t)m + 1, s));
    DBuf<unsigned char> tmp;
    tmp.alloc(bytes);
    GN_CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, poff.p, (int64_t)m + 1, s));
    count_launch();
    GN_CK(cudaMemcpyAsync(&K->npair, poff.p + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GN_CK(cudaStreamSynchronize(s));
  }
  // ---- M COO keys: [Hessian | pairs | diagonal] (condensed.hpp:44-74)
  const int64_t total = K->nh + K->npair + n;
  if (total > 0x7fffffffLL) throw Error(GN_ERR_INVALID, "condensed KKT: M COO exceeds int32");
  K->pka.alloc(K->npair + 1);
  K->pkb.alloc(K->npair + 1);
  K->arow.alloc(static_cast<size_t>(K->annz) + 1);
  {
    DBuf<uint64_t> key;
    key.alloc(total + 1);
    if (K->nh) { k_keys_hess<<<nblk(K->nh), 256, 0, s>>>(K->nh, hr, hc, (uint64_t)n, key.p); count_launch(); }
    if (m) {
      k_pairs<<<nblk(m, 128), 128, 0, s>>>(m, K->A.ptr.p, K->A.idx.p, poff.p, (uint64_t)n,
                                           key.p + K->nh, K->pka.p, K->pkb.p, K->arow.p);
      count_launch();
    }
    if (n) { k_keys_diag<<<nblk(n), 256, 0, s>>>(n, key.p + K->nh + K->npair); count_launch(); }
    compress_keys(key.p, total, n, n, K->M, s);
  }
  K->mnnz = K->M.nnz;
  K->dvals.alloc(static_cast<size_t>(m) + kGuard);
  K->mvals.alloc(static_cast<size_t>(K->mnnz) + kGuard);
  GN_CK(cudaMemsetAsync(K->mvals.p, 0, sizeof(double) * (K->mnnz + kGuard), s));
  GN_CK(cudaGetLastError());
  GN_CK(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------- assembly
// A[s] = 0 (+) J[k] over the slot's J entries in ascending k (scatter_values).
__global__ void __launch_bounds__(256) k_set_jac_generic(int32_t annz, const int32_t* __restrict__ seg,
                                                         const int32_t* __restrict__ src,
                                                         const int32_t* __restrict__ pick,
                                                         const double* __restrict__ J,
                                                         double* __restrict__ A) {
  const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= annz) return;
  double acc = 0.0;
  const int32_t i1 = seg[sl + 1];
  for (int32_t i = seg[sl]; i < i1; ++i) {
    const int32_t k = src[i];
    acc += J[pick ? pick[k] : k];
  }
  A[sl] = acc;
}

// M[s] = 0 (+) H[k]... (+) (d_r a_ka) a_kb ... (+) (dw + sx_i), contributors in COO order;
// d_r precomputed once per row (launch_dvec) instead of once per pair.
__global__ void __launch_bounds__(256) k_assemble_generic(
    int32_t mnnz, int64_t nh, int64_t npair, const int32_t* __restrict__ seg,
    const int32_t* __restrict__ src, const int32_t* __restrict__ hpick,
    const double* __restrict__ H, const int32_t* __restrict__ pka,
    const int32_t* __restrict__ pkb, const int32_t* __restrict__ arow,
    const double* __restrict__ A, const double* __restrict__ sx,
    const double* __restrict__ dv, double dw, double* __restrict__ M) {
  const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= mnnz) return;
  double acc = 0.0;
  const int32_t i1 = seg[sl + 1];
  for (int32_t i = seg[sl]; i < i1; ++i) {
    const int64_t c = src[i];
    if (c < nh) {
      acc += H[hpick ? hpick[c] : c];
    } else if (c < nh + npair) {
      const int64_t p = c - nh;
      const int32_t ka = pka[p], kb = pkb[p];
      const double va = dv[arow[ka]] * A[ka];  // condensed.hpp:126-129
      acc += va * A[kb];
    } else {
      acc += dw + sx[c - nh - npair];
    }
  }
  M[sl] = acc;
}

// Lifted values -> the full COO order (the OPF kernels index the callback layout); the
// slots of fixed variables are never read by them.
__global__ void k_scatter_pick(int64_t n, const int32_t* __restrict__ pick,
                               const double* __restrict__ in, double* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[pick[k]] = in[k];
}

static const double* to_full(gn_kkt* K, const double* lifted, bool jac) {
  const int64_t nl = jac ? K->nj : K->nh, nf = jac ? K->ctx->d.nj : K->ctx->d.nh;
  DBuf<double>& buf = jac ? K->jfull : K->hfull;
  if (buf.n < static_cast<size_t>(nf) + 1) buf.alloc(static_cast<size_t>(nf) + 1);
  if (nl) {
    KTimer kt("k_scatter_pick", K->stream);
    k_scatter_pick<<<nblk(nl), 256, 0, K->stream>>>(nl, jac ? K->ctx->jpick.p : K->ctx->hpick.p,
                                                     lifted, buf.p);
    count_launch();
  }
  return buf.p;
}

void kkt_set_jacobian(gn_kkt* K, const double* J, bool full) {
  if (!K->annz) return;
  if (K->algo != 1 && opf_kkt_ready(K))
    return opf_set_jacobian(K, full ? J : to_full(K, J, true));
  const int32_t* pick = full ? K->ctx->jpick.p : nullptr;
  KTimer kt("k_set_jac_generic", K->stream);
  k_set_jac_generic<<<nblk(K->annz), 256, 0, K->stream>>>(K->annz, K->A.seg.p, K->A.src.p, pick,
                                                          J, K->avals.p);
  count_launch();
  GN_CK(cudaGetLastError());
}

void kkt_assemble(gn_kkt* K, const double* H, const double* sx, const double* ss, double dw,
                  double dc, bool full) {
  if (!K->mnnz) return;
  if (K->algo != 1 && opf_kkt_ready(K))
    return opf_assemble(K, full ? H : to_full(K, H, false), sx, ss, dw, dc);
  const int32_t* hpick = full ? K->ctx->hpick.p : nullptr;
  launch_dvec(K, ss, dw, dc);
  KTimer kt("k_assemble_generic", K->stream);
  k_assemble_generic<<<nblk(K->mnnz), 256, 0, K->stream>>>(
      K->mnnz, K->nh, K->npair, K->M.seg.p, K->M.src.p, hpick, H, K->pka.p, K->pkb.p,
      K->arow.p, K->avals.p, sx, K->dvals.p, dw, K->mvals.p);
  count_launch();
  GN_CK(cudaGetLastError());
}

}  // namespace gnb
