#pragma once
#include "gn_kkt.cuh"

#include <algorithm>
#include <cstdlib>

namespace gnb {

// CTAs actually launched for `nvb` virtual CTAs: GRIDNLP_B200_GRID_CAP[_SETJAC|_LINE|_BUS] =
// resident CTAs per SM to allow (0 or unset: one CTA per virtual CTA, the plain grid).
// Grid of `nvb` virtual CTAs capped at `cap` resident CTAs per SM (0: one CTA per virtual
// CTA, the plain grid).  The cap of a KKT is set by gn_kkt_set_grid_cap; its default is
// the GRIDNLP_B200_GRID_CAP environment variable.
inline int grid_cap_default() {
  static const int cap = [] {
    const char* e = std::getenv("GRIDNLP_B200_GRID_CAP");
    return std::max(0, e ? std::atoi(e) : 0);
  }();
  return cap;
}
inline unsigned grid_cap(int64_t nvb, int cap) {
  if (cap <= 0) return (unsigned)nvb;
  return (unsigned)std::min<int64_t>(nvb, (int64_t)cap * 148);
}

// Column / row blocks of the lifted OPF variables, in variable order.
enum ColType { C_PG = 0, C_QG, C_P, C_Q, C_V, C_TH, C_TYPES };

// Small per-entity tables (L2-resident) that let one thread enumerate an M
// column's slots and each slot's contributors in the reference's summation
// order without any per-contributor index map.
struct OpfKktTab {
  int32_t T, N, L, G;
  int32_t bal_p0, bal_q0, flow_p0, flow_q0, therm0, ang0, ramp0;
  int64_t ho[K_COUNT], jo[K_COUNT];
  const int32_t* lent;                  // [2G+2L+2N] free-entity rank (lifted var = lent*T + t) or -1
  const int32_t* items;                 // (type << 28 | entity) of every free entity, in
                                        // network-locality order (key bus, type, entity)
  int32_t n_items, tchunks;             // one warp per (item, 32-period chunk)
  const int32_t *lf, *lt, *l_therm;     // [L]
  const int8_t* fpos;                   // [5L] flow-row positions of (p, v_f, v_t, th_f, th_t) or -1
  const int8_t* apos;                   // [2L] angle-row positions of (th_f, th_t) or -1
  const int32_t *lidx_to, *lidx_from;   // [L] rank of l among its bus's incident lines
  const int32_t *gbus, *ppos, *qpos, *g_ramp;  // [G]
  const int32_t *ngp, *ngq;             // [N] free pg / qg generators at the bus
  const int32_t *bl_ptr, *bl;           // [N+1] incident lines sorted by l: l<<1 | is_from
  const int32_t *bg_ptr, *bg;           // [N+1] generators at the bus, ascending
  const int32_t *nb_ptr, *nb;           // [N+1] incident lines sorted by (other bus, l): l<<1|is_from
  const int32_t *lnb_ptr, *lnb;         // [L+1] lines l' > l sharing a bus: (l' , shared-bus bits)
  const int32_t *rowptr, *colptr;       // CSR(A) / CSC(M) from the generic build
  // fused (recompute-from-x) path
  int32_t pg0, qg0, p0, q0, v0, th0;    // variable block offsets (full x)
  const double *lg, *lb, *c2;           // line G, B; generator c2
  const int32_t* th_line;               // [LT] line of each thermal slot
  const int32_t* nb_inc;                // [nb] index of the nb entry in the bus's bl list
  int32_t maxdeg;                       // max incident lines of a bus
  int32_t s_lo, R, prev, next;          // ramp steps of a period shard (OpfDims)
  int32_t n_owned;                      // lifted columns owned (next ghosts follow)
  int32_t grid_cap;                     // KKT kernels' resident CTAs per SM (0: uncapped)
  // fused line kernel descriptors
  const int4* ldesc0;                   // [L] (f, t, thermal slot or -1, flags: v/th free at
                                        //  min/max terminal bits 0-3, min==t bit 4, max==t bit 5)
  const int4* ldesc1;                   // [L] (lnb begin, lnb end, lifted p rank, lifted q rank)
  const int32_t* lnbx;                  // [lnb] l' << 4 | t(l') == max << 3 | t(l') == min << 2 | bits
  const int2* blx;                      // [bl] (l << 1 | is_from, other bus) per incident line
  const double2* blgb;                  // [bl] (G, B) per incident line
  const int32_t* bpos;                  // [bl] neighbour-slot offsets (register bus classes)
  const int32_t* rbase;                 // A row start at t = 0: bal_p[N] bal_q[N] flow_p[L]
                                        // flow_q[L] thermal[LT] angle[L] (row (e, t) = + t*len)
  const int2* lcb;                      // [L] M column start at t = 0 of p(l), q(l)
  const int32_t* bprog_ptr;             // [N+1] per-bus slot programs of the v(n)/th(n) columns
  const unsigned long long* bprog;      // (row entity << 35 | type << 32 | lane mask)
  double kdw, kdc;                      // delta_w, delta_c of the assembly in flight (dval)
};

// d_r of the fused kernels: read from the k_fz_dvec vector, or (GN_DV_INLINE, tuning builds)
// recomputed from sigma_s by each consumer -- `dv` is then sigma_s itself.
#ifndef GN_DV_INLINE
#define GN_DV_INLINE 0
#endif
#ifdef __CUDACC__
__device__ __forceinline__ double dval(const OpfKktTab& t, const double* __restrict__ dv,
                                       int64_t r) {
#if GN_DV_INLINE
  const double sd = dv[r] + t.kdw;  // condensed.hpp:112-116 (gn_opf_math.cuh dvec)
  const double c = 1.0 / (1.0 + t.kdc * sd);
  return sd * c;
#else
  return dv[r];
#endif
}
#endif

// Inputs of the fused (recompute-from-x) assembly.
struct FIn {
  const double* __restrict__ x;
  const double* __restrict__ w;
  double ow;
  const double* __restrict__ sx;
  const double* __restrict__ ss;
  double dw, dc;
};

// Bus-column kernel (v(n), th(n) columns): one warp per (bus, period chunk);
// lanes = (32/P periods) x (P incident-line slots), P = next pow2 >= degree.
// Bus-column kernel over one class of buses.  klass 0..kBusRegMax-1: buses of exactly
// klass+1 lines without parallel lines (line state in registers); klass kBusRegMax: the
// other buses of at most 8 lines (empty when GN_BUS3_MERGE), klass kBusRegMax+1: the rest
// (slot-program kernel, line state in shared memory sized by maxdeg).  Degree 7 joined the
// register classes in round 2 (case1354 x 24 -6%: its only slot-program buses were two of
// degree 7); 8 and 9 spill and measured slower than the slot program (9241 x 48 +2.4%).
void launch_fz_bus(const OpfKktTab& t, const int4* buses, int32_t n_buses, int32_t maxdeg,
                   int klass, const FIn& in, const double* dv, double* M, int32_t* rows,
                   int32_t* bad, cudaStream_t s);
#ifndef GN_BUS_REGMAX
#define GN_BUS_REGMAX 7  // register-resident classes d1..d<GN_BUS_REGMAX> (6..9; 8 and 9 spill)
#endif
constexpr int kBusRegMax = GN_BUS_REGMAX;
static_assert(kBusRegMax >= 6 && kBusRegMax <= 9, "register classes d1..d6 .. d1..d9");
// per bus: (n, bl begin, deg [| program length << 8], boff | program begin),
// (lifted v rank, lifted th rank, 0, 0), (M start of v(n, t=0), v column length,
// M start of th(n, t=0), th column length)
constexpr int kBusDesc = 3;
constexpr int kBusClasses = kBusRegMax + 2;
// descriptor int4s per bus of class k: the register classes (k < kBusRegMax, degree k + 1)
// also carry their lines inline -- (l << 1 | is_from, other bus, neighbour-slot offsets) and
// (G, B) per line -- so every load of a warp depends on its bus index only
__host__ __device__ constexpr int bus_desc_stride(int k) { return k < kBusRegMax ? kBusDesc + 2 * (k + 1) : kBusDesc; }
bool fz_bus_fits(int32_t maxdeg);  // one warp's shared memory fits (else: no fused path)

struct OpfKkt {
  bool ready = false;
  int32_t type_lo[C_TYPES + 1] = {};  // items of column type ty: [type_lo[ty], type_lo[ty+1])
  // fork/join of the column kernels over auxiliary streams (same priority as the KKT's)
  // aux[0 .. kBusClasses-1]: bus-class lanes; aux[kAuxSetJac]: set_jacobian beside assemble
  static constexpr int kAuxSetJac = kBusClasses, kAux = kBusClasses + 1;
  cudaStream_t aux[kAux] = {};
  cudaEvent_t ev_fork = nullptr, ev_fork2 = nullptr, ev_join[kAux] = {};
  int aux_prio = 0;
  ~OpfKkt() {
    for (auto& a : aux) if (a) cudaStreamDestroy(a);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_fork2) cudaEventDestroy(ev_fork2);
    for (auto& e : ev_join) if (e) cudaEventDestroy(e);
  }
  OpfKktTab t{};
  DBuf<int32_t> lent, items, lf, lt, l_therm, lidx_to, lidx_from, gbus, ppos, qpos, g_ramp, ngp,
      ngq, bl_ptr, bl, bg_ptr, bg, nb_ptr, nb, lnb_ptr, lnb, nb_inc;
  DBuf<int8_t> fpos, apos;
  bool fused_ready = false;
  DBuf<int32_t> lnbx;
  DBuf<int4> ldesc0, ldesc1;
  DBuf<int32_t> bprog_ptr;
  DBuf<unsigned long long> bprog;
  DBuf<int4> bus_cls[kBusClasses];  // bus descriptors by degree class (bus-column kernel)
  DBuf<int2> blx;
  DBuf<int32_t> bpos, rbase;
  DBuf<int2> lcb;
  int32_t maxdeg_rest = 0;
  DBuf<double2> blgb;
  int32_t n_bus_cls[kBusClasses] = {};
};


}  // namespace gnb
