// Period-shard halo over peer memory: the only data a period shard needs
// from its neighbours is the ramp coupling of opf.hpp:343-351 -- the boundary generator
// set-points pg(., t0 - 1) / pg(., t1) and the sigma_s of the boundary ramp rows (G doubles
// each) -- plus the one-double objective partial of every shard.
//
// Every rank owns a small device *region* (cudaMalloc, exported with cudaIpcGetMemHandle)
// that its neighbours write into with plain stores over NVLink / NVSwitch:
//
//   xprev[2][GR]  written by rank - 1: its pg(., last period)      -> our ghost pg(t0 - 1)
//   xnext[2][GR]  written by rank + 1: its pg(., first period)     -> our ghost pg(t1)
//   snext[2][GR]  written by rank + 1: sigma_s of its step-t0 rows -> our ghost ramp rows
//   fpart[2][W]   written by rank q:   its objective partial (slot q)
//   flags         step counters, released (st.release.sys) by the writer after its data
//
// One kernel per exchange (one CTA): pack and store into the neighbours' regions, fence,
// release the step flag; acquire-spin on our own flags; unpack into x / sigma_s.  Buffers
// alternate with the step parity; every rank's exchange both sends to and receives from
// each neighbour, so a writer can never run two steps ahead of a reader.  No host call,
// no NCCL: the whole step (callbacks, KKT and exchanges) is capturable in one CUDA graph.
// Ranks must run on different GPUs (a spin on one GPU waiting for another process's
// kernel is not guaranteed to make progress); on one GPU the protocol is exercised by
// gn_halo_exchange_emulated (all ranks in one cooperative launch) and the store path by
// separate SEND / RECV phases with a host barrier between them.
#include <cooperative_groups.h>

#include <cstring>
#include <vector>

#include "gn_internal.cuh"

namespace gnb {

constexpr int kHaloMaxWorld = 64;
constexpr int kHaloThreads = 256;

struct HaloView {       // everything the exchange kernel of one rank needs (by value)
  double* const* regions;  // [world] region base of every rank, as this process maps it
  int32_t rank, world, GR, prev, next;
  int64_t xprev, xnext, snext, fpart, flags;  // offsets (doubles / u64) inside a region
  const int32_t *pg_first, *pg_last, *g_prev, *g_next, *rows_first, *rows_ghost;
  unsigned long long* step;   // local counters: [0] halo, [1] objective
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait until *f >= s.  A peer that never arrives (a crashed rank, mismatched step counts)
// must not hang the GPU: after kHaloTimeoutNs the kernel traps, which fails this rank's
// context loudly instead of spinning forever.
constexpr unsigned long long kHaloTimeoutNs = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ void wait_flag(const unsigned long long* f, unsigned long long s) {
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_sys(f) < s) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > kHaloTimeoutNs) __trap();
  }
}
__device__ __forceinline__ unsigned long long* flag(double* region, const HaloView& h, int i) {
  return reinterpret_cast<unsigned long long*>(region + h.flags) + 16 * i;  // 128-byte apart
}
// flag slots: 0 = from prev, 1 = from next, 2 + q = objective of rank q

enum { PH_SEND = 1, PH_RECV = 2 };

__device__ void halo_body(const HaloView& h, double* __restrict__ x, double* __restrict__ ss,
                          int phase) {
  __shared__ unsigned long long s_step;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) s_step = (phase & PH_SEND) ? ++h.step[0] : h.step[0];
  __syncthreads();
  const unsigned long long s = s_step;
  const int64_t buf = (int64_t)(s & 1) * h.GR;
  double* mine = h.regions[h.rank];
  if (phase & PH_SEND) {
    if (h.next) {
      double* r = h.regions[h.rank + 1];
      for (int k = tid; k < h.GR; k += nt) r[h.xprev + buf + k] = x[h.pg_last[k]];
    }
    if (h.prev) {
      double* r = h.regions[h.rank - 1];
      for (int k = tid; k < h.GR; k += nt) {
        r[h.xnext + buf + k] = x[h.pg_first[k]];
        r[h.snext + buf + k] = ss[h.rows_first[k]];
      }
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) {
      if (h.next) st_release_sys(flag(h.regions[h.rank + 1], h, 0), s);
      if (h.prev) st_release_sys(flag(h.regions[h.rank - 1], h, 1), s);
    }
  }
  if (phase & PH_RECV) {
    if (tid == 0) {
      if (h.prev) wait_flag(flag(mine, h, 0), s);
      if (h.next) wait_flag(flag(mine, h, 1), s);
    }
    __syncthreads();
    for (int k = tid; k < h.GR; k += nt) {  // L2 reads (__ldcg): never a stale L1 line
      if (h.prev) x[h.g_prev[k]] = __ldcg(mine + h.xprev + buf + k);
      if (h.next) {
        x[h.g_next[k]] = __ldcg(mine + h.xnext + buf + k);
        ss[h.rows_ghost[k]] = __ldcg(mine + h.snext + buf + k);
      }
    }
  }
}

__device__ void fsum_body(const HaloView& h, const double* __restrict__ f_local,
                          double* __restrict__ f_global, int phase) {
  __shared__ unsigned long long s_step;
  const int tid = threadIdx.x;
  if (tid == 0) s_step = (phase & PH_SEND) ? ++h.step[1] : h.step[1];
  __syncthreads();
  const unsigned long long s = s_step;
  const int64_t buf = (int64_t)(s & 1) * kHaloMaxWorld;
  if ((phase & PH_SEND) && tid < h.world) {  // thread q: our partial into rank q's slot
    double* r = h.regions[tid];
    r[h.fpart + buf + h.rank] = f_local[0];
    st_release_sys(flag(r, h, 2 + h.rank), s);  // orders this thread's store before it
  }
  if (phase & PH_RECV) {
    double* mine = h.regions[h.rank];
    if (tid < h.world) wait_flag(flag(mine, h, 2 + tid), s);
    __syncthreads();
    if (tid == 0) {  // rank order: the same value on every rank, run to run
      double tot = __ldcg(mine + h.fpart + buf);
      for (int q = 1; q < h.world; ++q) tot += __ldcg(mine + h.fpart + buf + q);
      f_global[0] = tot;
    }
  }
}

__global__ void __launch_bounds__(kHaloThreads) k_halo(HaloView h, double* x, double* ss,
                                                      int phase) {
  halo_body(h, x, ss, phase);
}
__global__ void __launch_bounds__(kHaloThreads) k_halo_fsum(HaloView h, const double* f_local,
                                                           double* f_global, int phase) {
  fsum_body(h, f_local, f_global, phase);
}
// One-GPU emulation: every rank's exchange in one cooperative launch (CTA r = rank r), so
// the cross-rank spins are between co-resident CTAs of one kernel.
struct HaloAll {
  HaloView v[8];
  double* x[8];
  double* ss[8];
};
__global__ void __launch_bounds__(kHaloThreads) k_halo_emulated(HaloAll a) {
  halo_body(a.v[blockIdx.x], a.x[blockIdx.x], a.ss[blockIdx.x], PH_SEND | PH_RECV);
}

}  // namespace gnb

struct gn_halo {
  int device = 0;
  int32_t rank = 0, world = 1;
  gn_ctx* ctx = nullptr;
  size_t region_bytes = 0;
  double* region = nullptr;                 // ours (cudaMalloc: IPC-exportable)
  std::vector<double*> remote;              // host copy of the region table
  std::vector<bool> opened;                 // remote[q] came from cudaIpcOpenMemHandle
  gnb::DBuf<double*> regions;               // device copy of the region table
  gnb::DBuf<int32_t> idx;                   // pg_first pg_last g_prev g_next rows_first rows_ghost
  gnb::DBuf<unsigned long long> step;       // [halo, objective] counters
  gnb::HaloView view{};
  bool linked = false;
};

namespace {
int hfail(gn_error* err, int code, const char* msg) {
  if (err) {
    err->code = code;
    err->pattern = err->record = -1;
    std::snprintf(err->message, sizeof err->message, "%s", msg);
  }
  return code;
}
cudaStream_t sarg(void* s) { return static_cast<cudaStream_t>(s); }
void finish_view(gn_halo* h) {
  h->regions.alloc(h->remote.size());
  GN_CK(cudaMemcpy(h->regions.p, h->remote.data(), sizeof(double*) * h->remote.size(),
                   cudaMemcpyHostToDevice));
  h->view.regions = h->regions.p;
  h->linked = true;
}
}  // namespace

extern "C" {

int gn_halo_create(gn_ctx* c, int32_t rank, int32_t world, gn_halo** out, gn_error* err) {
  if (!c || !out) return hfail(err, GN_ERR_INVALID, "null argument");
  *out = nullptr;
  if (world < 1 || world > gnb::kHaloMaxWorld || rank < 0 || rank >= world)
    return hfail(err, GN_ERR_INVALID, "halo: rank / world out of range (world <= 64)");
  const gnb::OpfDims& d = c->d;
  if ((rank > 0) != (d.prev != 0) || (rank < world - 1) != (d.next != 0))
    return hfail(err, GN_ERR_INVALID, "halo: rank does not match the context's shard");
  gn_halo* h = nullptr;
  try {
    GN_CK(cudaSetDevice(c->device));
    h = new gn_halo();
    h->device = c->device;
    h->rank = rank;
    h->world = world;
    h->ctx = c;
    ++c->refs;
    const int32_t GR = d.GR;
    gnb::HaloView& v = h->view;
    v.rank = rank; v.world = world; v.GR = GR; v.prev = d.prev; v.next = d.next;
    v.xprev = 0;
    v.xnext = 2LL * GR;
    v.snext = 4LL * GR;
    v.fpart = 6LL * GR;
    v.flags = (v.fpart + 2LL * gnb::kHaloMaxWorld + 15) / 16 * 16;  // 128-byte aligned
    h->region_bytes = sizeof(double) * (v.flags + 16LL * (2 + gnb::kHaloMaxWorld));
    GN_CK(cudaMalloc(&h->region, h->region_bytes));
    GN_CK(cudaMemset(h->region, 0, h->region_bytes));
    std::vector<int32_t> ix(6 * static_cast<size_t>(GR) + 1, 0);
    for (int32_t k = 0; k < GR; ++k) {
      const int32_t g = c->ramp_gens[k];
      ix[0 * GR + k] = d.pg0 + g * d.T;                     // pg(., first period)
      ix[1 * GR + k] = d.pg0 + g * d.T + d.T - 1;           // pg(., last period)
      ix[2 * GR + k] = d.gh_prev + k;                       // ghost pg(t0 - 1)
      ix[3 * GR + k] = d.gh_next + k;                       // ghost pg(t1)
      ix[4 * GR + k] = d.ramp0 + k * d.R;                   // our rows of step t0
      ix[5 * GR + k] = d.ramp0 + k * d.R + (d.T - d.s_lo);  // ghost rows of step t1
    }
    h->idx.alloc(ix.size());
    GN_CK(cudaMemcpy(h->idx.p, ix.data(), sizeof(int32_t) * ix.size(), cudaMemcpyHostToDevice));
    v.pg_first = h->idx.p; v.pg_last = h->idx.p + GR; v.g_prev = h->idx.p + 2 * GR;
    v.g_next = h->idx.p + 3 * GR; v.rows_first = h->idx.p + 4 * GR; v.rows_ghost = h->idx.p + 5 * GR;
    h->step.alloc(2);
    GN_CK(cudaMemset(h->step.p, 0, 2 * sizeof(unsigned long long)));
    v.step = h->step.p;
    h->remote.assign(world, nullptr);
    h->opened.assign(world, false);
    h->remote[rank] = h->region;
    *out = h;
    if (err) { err->code = GN_OK; err->message[0] = 0; }
    return GN_OK;
  } catch (const gnb::Error& e) {
    if (h) gn_halo_destroy(h);
    return hfail(err, e.code, e.what());
  }
}

int gn_halo_ipc_handle(gn_halo* h, void* handle) {
  if (!h || !handle) return GN_ERR_INVALID;
  try {
    GN_CK(cudaSetDevice(h->device));
    cudaIpcMemHandle_t m;
    GN_CK(cudaIpcGetMemHandle(&m, h->region));
    std::memcpy(handle, &m, sizeof m);
    return GN_OK;
  } catch (const gnb::Error& e) {
    return e.code;
  }
}

int gn_halo_open(gn_halo* h, const void* handles) {
  if (!h || !handles || h->linked) return GN_ERR_INVALID;
  try {
    GN_CK(cudaSetDevice(h->device));
    const auto* b = static_cast<const unsigned char*>(handles);
    for (int32_t q = 0; q < h->world; ++q) {
      if (q == h->rank) continue;
      cudaIpcMemHandle_t m;
      std::memcpy(&m, b + static_cast<size_t>(q) * GN_HALO_HANDLE_BYTES, sizeof m);
      void* p = nullptr;
      GN_CK(cudaIpcOpenMemHandle(&p, m, cudaIpcMemLazyEnablePeerAccess));
      h->remote[q] = static_cast<double*>(p);
      h->opened[q] = true;
    }
    finish_view(h);
    return GN_OK;
  } catch (const gnb::Error& e) {
    return e.code;
  }
}

int gn_halo_link(gn_halo* const* halos, int32_t world) {
  if (!halos || world < 1) return GN_ERR_INVALID;
  for (int32_t q = 0; q < world; ++q)
    if (!halos[q] || halos[q]->world != world || halos[q]->rank != q || halos[q]->linked)
      return GN_ERR_INVALID;
  try {
    for (int32_t r = 0; r < world; ++r) {
      GN_CK(cudaSetDevice(halos[r]->device));
      for (int32_t q = 0; q < world; ++q) halos[r]->remote[q] = halos[q]->region;
      finish_view(halos[r]);
    }
    return GN_OK;
  } catch (const gnb::Error& e) {
    return e.code;
  }
}

int gn_halo_exchange(gn_halo* h, double* x, double* sigma_s, int phase, void* stream) {
  if (!h || !h->linked || !x || !sigma_s || phase < 1 || phase > 3) return GN_ERR_INVALID;
  try {
    GN_CK(cudaSetDevice(h->device));
    if (h->view.GR > 0 && (h->view.prev || h->view.next)) {
      gnb::KTimer kt("k_halo", sarg(stream));
      gnb::k_halo<<<1, gnb::kHaloThreads, 0, sarg(stream)>>>(h->view, x, sigma_s, phase);
      gnb::count_launch();
      GN_CK(cudaGetLastError());
    }
    return GN_OK;
  } catch (const gnb::Error& e) {
    return e.code;
  }
}

int gn_halo_objective(gn_halo* h, const double* f_local, double* f_global, int phase,
                      void* stream) {
  if (!h || !h->linked || !f_local || !f_global || phase < 1 || phase > 3) return GN_ERR_INVALID;
  try {
    GN_CK(cudaSetDevice(h->device));
    gnb::KTimer kt("k_halo_fsum", sarg(stream));
    gnb::k_halo_fsum<<<1, gnb::kHaloThreads, 0, sarg(stream)>>>(h->view, f_local, f_global, phase);
    gnb::count_launch();
    GN_CK(cudaGetLastError());
    return GN_OK;
  } catch (const gnb::Error& e) {
    return e.code;
  }
}

int gn_halo_exchange_emulated(gn_halo* const* halos, int32_t world, double* const* xs,
                              double* const* ss, void* stream) {
  if (!halos || !xs || !ss || world < 1 || world > 8) return GN_ERR_INVALID;
  gnb::HaloAll a{};
  for (int32_t q = 0; q < world; ++q) {
    if (!halos[q] || !halos[q]->linked || halos[q]->device != halos[0]->device ||
        halos[q]->rank != q)
      return GN_ERR_INVALID;
    a.v[q] = halos[q]->view;
    a.x[q] = xs[q];
    a.ss[q] = ss[q];
  }
  try {
    GN_CK(cudaSetDevice(halos[0]->device));
    void* args[] = {&a};
    GN_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(gnb::k_halo_emulated),
                                      dim3(world), dim3(gnb::kHaloThreads), args, 0, sarg(stream)));
    gnb::count_launch();
    return GN_OK;
  } catch (const gnb::Error& e) {
    return e.code;
  }
}

int gn_halo_destroy(gn_halo* h) {
  if (!h) return GN_OK;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (int32_t q = 0; q < h->world; ++q)
    if (h->opened.size() > static_cast<size_t>(q) && h->opened[q]) cudaIpcCloseMemHandle(h->remote[q]);
  if (h->region) cudaFree(h->region);
  gn_ctx* c = h->ctx;
  delete h;
  if (c) gnb::ctx_unref(c);
  return GN_OK;
}

}  // extern "C"
