#pragma once
#include "gn_eval.cuh"

namespace gnb {

struct OpfKkt;
// doubles allocated after A / M / d values: a guard band that no kernel may touch
// (gn_debug_kkt_guard fills and checks it)
constexpr int64_t kGuard = 512;

// A compressed (CSC-ordered) pattern plus its scatter/gather maps.
struct Csc {
  int32_t nnz = 0;
  DBuf<int32_t> ptr;   // [ncols + 1]
  DBuf<int32_t> idx;   // [nnz] row index per slot
  DBuf<int32_t> seg;   // [nnz + 1] first sorted position of each slot
  DBuf<int32_t> src;   // [coo] COO index at each sorted position (contributor lists)
  DBuf<int32_t> slot;  // [coo] slot_map: compressed slot of each COO entry
};

// Sort 64-bit (col * nrows + row) keys and compress (matrix.hpp:45-81).  keys is clobbered.
void compress_keys(uint64_t* keys, int64_t nnz, int32_t nrows, int32_t ncols, Csc& out,
                   cudaStream_t s);

}  // namespace gnb

struct gn_kkt {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t owned_stream = nullptr;  // created here; destroyed with the object
  int refs = 0;         // live objects built on this one (KKTs / IPMs)
  bool closed = false;  // destroy requested; freed when refs drops to 0
  gn_ctx* ctx = nullptr;  // set for gn_kkt_create_lifted
  int32_t n = 0, m = 0;
  int64_t nj = 0, nh = 0, npair = 0;
  int32_t annz = 0, mnnz = 0;
  int algo = 0;
  gnb::Csc A;                    // CSR(A) (as CSC of A^T): ptr = rowptr, idx = colidx, slot = jac_slots
  gnb::Csc M;                    // M lower CSC: ptr = colptr, idx = rowidx, slot = [hess|pair|diag]
  gnb::DBuf<int32_t> pka, pkb;   // per pair: CSR positions ka, kb
  gnb::DBuf<int32_t> arow;       // per CSR(A) entry: its row
  gnb::DBuf<double> avals, mvals, dvals;
  gnb::DBuf<double> sj, sh, ssx, sss;  // host-mode staging
  gnb::DBuf<double> jfull, hfull;      // lifted inputs scattered to the full COO order (OPF kernels)
  gnb::OpfKkt* opf = nullptr;    // OPF-specialised tables (gn_kkt_create_lifted)
  // gn_kkt_values_start: the read-back on a side stream, ordered before the next write
  cudaStream_t vstream = nullptr;
  cudaEvent_t vstart = nullptr, vdone = nullptr;
  bool vpend_a = false, vpend_m = false;  // which arrays the side-stream copy still reads
};

namespace gnb {
void kkt_build(gn_kkt* K, const int32_t* jr, const int32_t* jc, const int32_t* hr,
               const int32_t* hc);
void kkt_set_jacobian(gn_kkt* K, const double* J, bool full);
void kkt_assemble(gn_kkt* K, const double* H, const double* sx, const double* ss, double dw,
                  double dc, bool full);
bool opf_kkt_prepare(gn_kkt* K);
// *diff += number of positions where a[i] != b[i]
void count_diff(const int32_t* a, const int32_t* b, int64_t n, int32_t* diff, cudaStream_t s);
// d_r = (sigma_s + dw) / (1 + dc (sigma_s + dw)) per row into K->dvals (condensed.hpp:111-116),
// in the reference's operation order: every consumer reads it instead of dividing again.
void launch_dvec(gn_kkt* K, const double* ss, double dw, double dc);
void opf_kkt_free(gn_kkt* K);
void opf_set_grid_cap(gn_kkt* K, int ctas_per_sm);
bool opf_kkt_ready(const gn_kkt* K);
bool opf_fused_ready(const gn_kkt* K);
bool opf_fused_verify(gn_kkt* K);
void opf_set_jacobian_fused(gn_kkt* K, const double* x);
void opf_update_fused(gn_kkt* K, const double* x, const double* w, double ow, const double* sx,
                      const double* ss, double dw, double dc);
void opf_assemble_fused(gn_kkt* K, const double* x, const double* w, double ow, const double* sx,
                        const double* ss, double dw, double dc);
void opf_set_jacobian(gn_kkt* K, const double* Jfull);
void opf_assemble(gn_kkt* K, const double* Hfull, const double* sx, const double* ss, double dw,
                  double dc);
// Does a published context's lifted structure equal this COO (device arrays)?  Returns it.
gn_ctx* find_published(int device, int32_t n, int32_t m, int64_t nj, const int32_t* jr,
                       const int32_t* jc, int64_t nh, const int32_t* hr, const int32_t* hc,
                       cudaStream_t s);
}  // namespace gnb
