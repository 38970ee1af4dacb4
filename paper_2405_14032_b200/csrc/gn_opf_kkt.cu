// OPF-specialised condensed-KKT kernels (FULL J/H inputs).
//
// set_jacobian: one thread per A row (row-major = entity-major, t fastest):
//   the J record(s) of the row are read and written at rowptr[r] + position.
// assemble: one thread per M column (lifted var = (entity, t)); the thread walks
//   the network topology and adds every contributor of every slot of its column
//   in exactly the order CondensedKkt::assemble visits them
//   (condensed.hpp:118-134: 0 (+) H in COO order (+) AtDA pairs in row order
//   (+) dw + sigma_x), so M is bit-identical to the generic
//   contributor-list kernel and to the reference for equal inputs — with no
//   per-contributor index maps (only per-entity tables, which stay in L2).
//   CTAs are ordered period-major so the H/A/sigma working set of the periods
//   in flight (~15 MB each at 30k buses) stays in the 126 MB L2.
//
// The enumeration is checked against the generic structure once at setup
// (opf_kkt_prepare): if any column's rows differ, the specialised path is
// disabled and the generic kernels are used.
#include <algorithm>
#include <cstring>
#include <numeric>

#include <type_traits>

#include "gn_opf_kkt.cuh"

namespace gnb {

// one slot-program launch for every bus the register classes do not take (parallel lines,
// degree > 6): its ~20 us latency floor is paid once, not per class (0: <= 8 / rest split)
#ifndef GN_BUS3_MERGE
#define GN_BUS3_MERGE 1
#endif

constexpr int kMB = 128;  // threads (columns) per CTA

struct In {
  const double* __restrict__ H;
  const double* __restrict__ A;
  const double* __restrict__ sx;
  const double* __restrict__ dv;  // d_r per row (launch_dvec, condensed.hpp:112-116)
  double dw;
};

__device__ __forceinline__ double pairval(const OpfKktTab& t, const In& in, int32_t r, int ia,
                                          int ib) {
  const int32_t rp = __ldg(t.rowptr + r);
  const double va = in.dv[r] * in.A[rp + ia];  // condensed.hpp:126-129
  return va * in.A[rp + ib];
}

__device__ __forceinline__ int32_t lidx(const OpfKktTab& t, int32_t l, int32_t b) {
  return b == __ldg(t.lt + l) ? __ldg(t.lidx_to + l) : __ldg(t.lidx_from + l);
}

__device__ __forceinline__ bool freev(const OpfKktTab& t, int type, int32_t e) {
  int32_t off;
  switch (type) {
    case C_PG: off = 0; break;
    case C_QG: off = t.G; break;
    case C_P: off = 2 * t.G; break;
    case C_Q: off = 2 * t.G + t.L; break;
    case C_V: off = 2 * t.G + 2 * t.L; break;
    default: off = 2 * t.G + 2 * t.L + t.N; break;
  }
  return __ldg(t.lent + off + e) >= 0;
}

// Writes (value or row index) of one slot.
template <bool STRUCT>
struct Out {
  double* M;
  int32_t* rows;
  int64_t base;
  int j = 0;
  __device__ __forceinline__ void put(double v, int32_t row) {
    if constexpr (STRUCT) rows[base + j] = row; else M[base + j] = v;
    ++j;
  }
};

__device__ __forceinline__ int32_t lv(const OpfKktTab& t, int type, int32_t e, int32_t tt) {
  int32_t off;
  switch (type) {
    case C_PG: off = 0; break;
    case C_QG: off = t.G; break;
    case C_P: off = 2 * t.G; break;
    case C_Q: off = 2 * t.G + t.L; break;
    case C_V: off = 2 * t.G + 2 * t.L; break;
    default: off = 2 * t.G + 2 * t.L + t.N; break;
  }
  const int32_t k = __ldg(t.lent + off + e);
  return k < 0 ? -1 : k * t.T + tt;
}

// ------------------------------------------------------------- M columns
template <bool STRUCT>
__device__ void col_th(const OpfKktTab& t, const In& in, int32_t n, int32_t tt, Out<STRUCT>& o) {
  const int32_t T = t.T;
  const int32_t b0 = __ldg(t.bl_ptr + n), b1 = __ldg(t.bl_ptr + n + 1);
  const int32_t me = lv(t, C_TH, n, tt);
  {  // diagonal
    double acc = 0.0;
    if constexpr (!STRUCT) {
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        acc += in.H[t.ho[K_FLOW_P] + 15 * ((int64_t)l * T + tt) + (fr ? 12 : 14)];
      }
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        acc += in.H[t.ho[K_FLOW_Q] + 15 * ((int64_t)l * T + tt) + (fr ? 12 : 14)];
      }
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        acc += in.H[t.ho[K_ANGLE] + 3 * ((int64_t)l * T + tt) + (fr ? 0 : 2)];
      }
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        const int p = __ldg(t.fpos + 5 * l + (fr ? 3 : 4));
        acc += pairval(t, in, t.flow_p0 + l * T + tt, p, p);
      }
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        const int p = __ldg(t.fpos + 5 * l + (fr ? 3 : 4));
        acc += pairval(t, in, t.flow_q0 + l * T + tt, p, p);
      }
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        const int p = __ldg(t.apos + 2 * l + (fr ? 0 : 1));
        acc += pairval(t, in, t.ang0 + l * T + tt, p, p);
      }
      acc += in.dw + in.sx[me];
    }
    o.put(acc, me);
  }
  // th(n') for neighbours n' > n, lines grouped by neighbour (ascending l)
  const int32_t q0 = __ldg(t.nb_ptr + n), q1 = __ldg(t.nb_ptr + n + 1);
  int32_t i = q0;
  while (i < q1) {
    const int32_t e0 = __ldg(t.nb + i), l0 = e0 >> 1;
    const int32_t nb = (e0 & 1) ? __ldg(t.lt + l0) : __ldg(t.lf + l0);
    int32_t k = i + 1;
    while (k < q1) {
      const int32_t ek = __ldg(t.nb + k), lk = ek >> 1;
      const int32_t bk = (ek & 1) ? __ldg(t.lt + lk) : __ldg(t.lf + lk);
      if (bk != nb) break;
      ++k;
    }
    if (nb > n && freev(t, C_TH, nb)) {
      double acc = 0.0;
      if constexpr (!STRUCT) {
        for (int32_t u = i; u < k; ++u) {
          const int32_t l = __ldg(t.nb + u) >> 1;
          acc += in.H[t.ho[K_FLOW_P] + 15 * ((int64_t)l * T + tt) + 13];
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t l = __ldg(t.nb + u) >> 1;
          acc += in.H[t.ho[K_FLOW_Q] + 15 * ((int64_t)l * T + tt) + 13];
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t l = __ldg(t.nb + u) >> 1;
          acc += in.H[t.ho[K_ANGLE] + 3 * ((int64_t)l * T + tt) + 1];
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          const int pa = __ldg(t.fpos + 5 * l + (fr ? 4 : 3)), pb = __ldg(t.fpos + 5 * l + (fr ? 3 : 4));
          acc += pairval(t, in, t.flow_p0 + l * T + tt, pa, pb);
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          const int pa = __ldg(t.fpos + 5 * l + (fr ? 4 : 3)), pb = __ldg(t.fpos + 5 * l + (fr ? 3 : 4));
          acc += pairval(t, in, t.flow_q0 + l * T + tt, pa, pb);
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          const int pa = __ldg(t.apos + 2 * l + (fr ? 1 : 0)), pb = __ldg(t.apos + 2 * l + (fr ? 0 : 1));
          acc += pairval(t, in, t.ang0 + l * T + tt, pa, pb);
        }
      }
      o.put(acc, lv(t, C_TH, nb, tt));
    }
    i = k;
  }
}

template <bool STRUCT>
__device__ void col_v(const OpfKktTab& t, const In& in, int32_t n, int32_t tt, Out<STRUCT>& o) {
  const int32_t T = t.T;
  const int32_t b0 = __ldg(t.bl_ptr + n), b1 = __ldg(t.bl_ptr + n + 1);
  const int32_t me = lv(t, C_V, n, tt);
  {  // diagonal (v, v): flow_p slot (1,1) or (2,2), flow_q likewise, pairs, diag
    double acc = 0.0;
    if constexpr (!STRUCT) {
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        acc += in.H[t.ho[K_FLOW_P] + 15 * ((int64_t)l * T + tt) + (fr ? 5 : 9)];
      }
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        acc += in.H[t.ho[K_FLOW_Q] + 15 * ((int64_t)l * T + tt) + (fr ? 5 : 9)];
      }
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        const int p = __ldg(t.fpos + 5 * l + (fr ? 1 : 2));
        acc += pairval(t, in, t.flow_p0 + l * T + tt, p, p);
      }
      for (int32_t i = b0; i < b1; ++i) {
        const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
        const int p = __ldg(t.fpos + 5 * l + (fr ? 1 : 2));
        acc += pairval(t, in, t.flow_q0 + l * T + tt, p, p);
      }
      acc += in.dw + in.sx[me];
    }
    o.put(acc, me);
  }
  const int32_t q0 = __ldg(t.nb_ptr + n), q1 = __ldg(t.nb_ptr + n + 1);
  // v(n') for neighbours n' > n
  for (int32_t i = q0; i < q1;) {
    const int32_t e0 = __ldg(t.nb + i), l0 = e0 >> 1;
    const int32_t nb = (e0 & 1) ? __ldg(t.lt + l0) : __ldg(t.lf + l0);
    int32_t k = i + 1;
    while (k < q1) {
      const int32_t ek = __ldg(t.nb + k), lk = ek >> 1;
      if (((ek & 1) ? __ldg(t.lt + lk) : __ldg(t.lf + lk)) != nb) break;
      ++k;
    }
    if (nb > n && freev(t, C_V, nb)) {
      double acc = 0.0;
      if constexpr (!STRUCT) {
        for (int32_t u = i; u < k; ++u) {
          const int32_t l = __ldg(t.nb + u) >> 1;
          acc += in.H[t.ho[K_FLOW_P] + 15 * ((int64_t)l * T + tt) + 6];
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t l = __ldg(t.nb + u) >> 1;
          acc += in.H[t.ho[K_FLOW_Q] + 15 * ((int64_t)l * T + tt) + 6];
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          const int pa = __ldg(t.fpos + 5 * l + (fr ? 2 : 1)), pb = __ldg(t.fpos + 5 * l + (fr ? 1 : 2));
          acc += pairval(t, in, t.flow_p0 + l * T + tt, pa, pb);
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          const int pa = __ldg(t.fpos + 5 * l + (fr ? 2 : 1)), pb = __ldg(t.fpos + 5 * l + (fr ? 1 : 2));
          acc += pairval(t, in, t.flow_q0 + l * T + tt, pa, pb);
        }
      }
      o.put(acc, lv(t, C_V, nb, tt));
    }
    i = k;
  }
  // th(x) for x in {n} U neighbours, ascending x
  bool self_done = false;
  for (int32_t i = q0; i <= q1;) {
    int32_t nb = 0x7fffffff, k = i + 1;
    if (i < q1) {
      const int32_t e0 = __ldg(t.nb + i), l0 = e0 >> 1;
      nb = (e0 & 1) ? __ldg(t.lt + l0) : __ldg(t.lf + l0);
      while (k < q1) {
        const int32_t ek = __ldg(t.nb + k), lk = ek >> 1;
        if (((ek & 1) ? __ldg(t.lt + lk) : __ldg(t.lf + lk)) != nb) break;
        ++k;
      }
    }
    if (!self_done && n < nb) {  // the (th(n), v(n)) slot: every incident line
      self_done = true;
      if (b1 > b0 && freev(t, C_TH, n)) {  // (an isolated bus has no such entry)
        double acc = 0.0;
        if constexpr (!STRUCT) {
          for (int32_t u = b0; u < b1; ++u) {
            const int32_t e = __ldg(t.bl + u), l = e >> 1, fr = e & 1;
            acc += in.H[t.ho[K_FLOW_P] + 15 * ((int64_t)l * T + tt) + (fr ? 7 : 11)];
          }
          for (int32_t u = b0; u < b1; ++u) {
            const int32_t e = __ldg(t.bl + u), l = e >> 1, fr = e & 1;
            acc += in.H[t.ho[K_FLOW_Q] + 15 * ((int64_t)l * T + tt) + (fr ? 7 : 11)];
          }
          for (int32_t u = b0; u < b1; ++u) {
            const int32_t e = __ldg(t.bl + u), l = e >> 1, fr = e & 1;
            const int pa = __ldg(t.fpos + 5 * l + (fr ? 3 : 4)), pb = __ldg(t.fpos + 5 * l + (fr ? 1 : 2));
            acc += pairval(t, in, t.flow_p0 + l * T + tt, pa, pb);
          }
          for (int32_t u = b0; u < b1; ++u) {
            const int32_t e = __ldg(t.bl + u), l = e >> 1, fr = e & 1;
            const int pa = __ldg(t.fpos + 5 * l + (fr ? 3 : 4)), pb = __ldg(t.fpos + 5 * l + (fr ? 1 : 2));
            acc += pairval(t, in, t.flow_q0 + l * T + tt, pa, pb);
          }
        }
        o.put(acc, lv(t, C_TH, n, tt));
      }
      continue;  // re-examine the same neighbour group
    }
    if (i >= q1) break;
    if (freev(t, C_TH, nb)) {  // (th(n'), v(n)): slot (4,1) if n is from, (3,2) if n is to
      double acc = 0.0;
      if constexpr (!STRUCT) {
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          acc += in.H[t.ho[K_FLOW_P] + 15 * ((int64_t)l * T + tt) + (fr ? 8 : 10)];
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          acc += in.H[t.ho[K_FLOW_Q] + 15 * ((int64_t)l * T + tt) + (fr ? 8 : 10)];
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          const int pa = __ldg(t.fpos + 5 * l + (fr ? 4 : 3)), pb = __ldg(t.fpos + 5 * l + (fr ? 1 : 2));
          acc += pairval(t, in, t.flow_p0 + l * T + tt, pa, pb);
        }
        for (int32_t u = i; u < k; ++u) {
          const int32_t e = __ldg(t.nb + u), l = e >> 1, fr = e & 1;
          const int pa = __ldg(t.fpos + 5 * l + (fr ? 4 : 3)), pb = __ldg(t.fpos + 5 * l + (fr ? 1 : 2));
          acc += pairval(t, in, t.flow_q0 + l * T + tt, pa, pb);
        }
      }
      o.put(acc, lv(t, C_TH, nb, tt));
    }
    i = k;
  }
}

// p(l) (Q = false) or q(l) (Q = true) columns.
template <bool STRUCT, bool Q>
__device__ void col_flow(const OpfKktTab& t, const In& in, int32_t l, int32_t tt, Out<STRUCT>& o) {
  const int32_t T = t.T;
  const int64_t r = (int64_t)l * T + tt;
  const int32_t f = __ldg(t.lf + l), to = __ldg(t.lt + l);
  const int32_t blo = min(f, to), bhi = max(f, to);
  const int32_t k = __ldg(t.l_therm + l);
  const int kb = Q ? K_BAL_Q_FLOW : K_BAL_P_FLOW, kf = Q ? K_FLOW_Q : K_FLOW_P;
  const int32_t bal0 = Q ? t.bal_q0 : t.bal_p0, flow0 = Q ? t.flow_q0 : t.flow_p0;
  const int32_t* ng = Q ? t.ngq : t.ngp;
  const int32_t me = lv(t, Q ? C_Q : C_P, l, tt);
  {
    double acc = 0.0;
    if constexpr (!STRUCT) {
      acc += in.H[t.ho[kb] + 2 * r];      // to-record (p,p)
      acc += in.H[t.ho[kb] + 2 * r + 1];  // from-record
      acc += in.H[t.ho[kf] + 15 * r];     // flow definition (0,0)
      if (k >= 0) acc += in.H[t.ho[K_THERMAL] + 3 * ((int64_t)k * T + tt) + (Q ? 2 : 0)];
      const int pl = __ldg(ng + blo) + lidx(t, l, blo);
      acc += pairval(t, in, bal0 + blo * T + tt, pl, pl);
      const int ph = __ldg(ng + bhi) + lidx(t, l, bhi);
      acc += pairval(t, in, bal0 + bhi * T + tt, ph, ph);
      acc += pairval(t, in, flow0 + (int32_t)r, 0, 0);
      if (k >= 0) acc += pairval(t, in, t.therm0 + k * T + tt, Q ? 1 : 0, Q ? 1 : 0);
      acc += in.dw + in.sx[me];
    }
    o.put(acc, me);
  }
  // flows l' > l sharing a bus (balance-row pairs, shared buses ascending)
  const int32_t a0 = __ldg(t.lnb_ptr + l), a1 = __ldg(t.lnb_ptr + l + 1);
  for (int32_t i = a0; i < a1; ++i) {
    const int32_t e = __ldg(t.lnb + i), l2 = e >> 2, bits = e & 3;
    double acc = 0.0;
    if constexpr (!STRUCT) {
      if (bits & 1) {
        const int pa = __ldg(ng + blo) + lidx(t, l2, blo), pb = __ldg(ng + blo) + lidx(t, l, blo);
        acc += pairval(t, in, bal0 + blo * T + tt, pa, pb);
      }
      if (bits & 2) {
        const int pa = __ldg(ng + bhi) + lidx(t, l2, bhi), pb = __ldg(ng + bhi) + lidx(t, l, bhi);
        acc += pairval(t, in, bal0 + bhi * T + tt, pa, pb);
      }
    }
    o.put(acc, lv(t, Q ? C_Q : C_P, l2, tt));
  }
  if (!Q && k >= 0) {  // (q(l), p(l)) from the thermal row
    double acc = 0.0;
    if constexpr (!STRUCT) {
      acc += in.H[t.ho[K_THERMAL] + 3 * ((int64_t)k * T + tt) + 1];
      acc += pairval(t, in, t.therm0 + k * T + tt, 1, 0);
    }
    o.put(acc, lv(t, C_Q, l, tt));
  }
  // v(b), then th(b), b ascending in {f, to}
#pragma unroll
  for (int blk = 0; blk < 2; ++blk) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int32_t b = s == 0 ? blo : bhi;
      const bool isf = (b == f);
      const int field = blk == 0 ? (isf ? 1 : 2) : (isf ? 3 : 4);
      const int pa = __ldg(t.fpos + 5 * l + field);
      if (pa < 0) continue;
      double acc = 0.0;
      if constexpr (!STRUCT) {
        acc += in.H[t.ho[kf] + 15 * r + field];  // local slot (field, 0)
        acc += pairval(t, in, flow0 + (int32_t)r, pa, 0);
      }
      o.put(acc, lv(t, blk == 0 ? C_V : C_TH, b, tt));
    }
  }
}

// pg(g) (Q = false) or qg(g) (Q = true) columns.
template <bool STRUCT, bool Q>
__device__ void col_gen(const OpfKktTab& t, const In& in, int32_t g, int32_t tt, Out<STRUCT>& o) {
  const int32_t T = t.T;
  const int32_t b = __ldg(t.gbus + g);
  const int32_t* pos = Q ? t.qpos : t.ppos;
  const int32_t* ng = Q ? t.ngq : t.ngp;
  const int32_t bal0 = Q ? t.bal_q0 : t.bal_p0;
  const int32_t rb = bal0 + b * T + tt;
  const int my = __ldg(pos + g);
  const int32_t kr = Q ? -1 : __ldg(t.g_ramp + g);
  const int32_t me = lv(t, Q ? C_QG : C_PG, g, tt);
  const int64_t r = (int64_t)g * T + tt;
  {
    double acc = 0.0;
    if constexpr (!STRUCT) {
      if (!Q) acc += in.H[t.ho[K_COST] + r];
      acc += in.H[t.ho[Q ? K_BAL_Q_INJ : K_BAL_P_INJ] + r];
      if (kr >= 0 && tt >= 1) acc += in.H[t.ho[K_RAMP] + 3 * ((int64_t)kr * (T - 1) + tt - 1)];
      if (kr >= 0 && tt + 1 < T) acc += in.H[t.ho[K_RAMP] + 3 * ((int64_t)kr * (T - 1) + tt) + 2];
      acc += pairval(t, in, rb, my, my);
      if (kr >= 0 && tt >= 1) acc += pairval(t, in, t.ramp0 + kr * (T - 1) + tt - 1, 1, 1);
      if (kr >= 0 && tt + 1 < T) acc += pairval(t, in, t.ramp0 + kr * (T - 1) + tt, 0, 0);
      acc += in.dw + in.sx[me];
    }
    o.put(acc, me);
  }
  if (kr >= 0 && tt + 1 < T) {  // (pg(g,t+1), pg(g,t))
    double acc = 0.0;
    if constexpr (!STRUCT) {
      acc += in.H[t.ho[K_RAMP] + 3 * ((int64_t)kr * (T - 1) + tt) + 1];
      acc += pairval(t, in, t.ramp0 + kr * (T - 1) + tt, 1, 0);
    }
    o.put(acc, me + 1);
  }
  // later generators at the same bus
  const int32_t g0 = __ldg(t.bg_ptr + b), g1 = __ldg(t.bg_ptr + b + 1);
  for (int32_t i = g0; i < g1; ++i) {
    const int32_t g2 = __ldg(t.bg + i);
    if (g2 <= g || !freev(t, Q ? C_QG : C_PG, g2)) continue;
    double acc = 0.0;
    if constexpr (!STRUCT) acc += pairval(t, in, rb, __ldg(pos + g2), my);
    o.put(acc, lv(t, Q ? C_QG : C_PG, g2, tt));
  }
  // incident flows
  const int32_t b0 = __ldg(t.bl_ptr + b), b1 = __ldg(t.bl_ptr + b + 1);
  const int nfree = __ldg(ng + b);
  for (int32_t i = b0; i < b1; ++i) {
    const int32_t l = __ldg(t.bl + i) >> 1;
    double acc = 0.0;
    if constexpr (!STRUCT) acc += pairval(t, in, rb, nfree + (i - b0), my);
    o.put(acc, lv(t, Q ? C_Q : C_P, l, tt));
  }
}

// One warp per (entity, 32 consecutive periods): control flow and the per-entity
// table reads are warp-uniform; sigma, rowptr and the M columns of the warp are
// contiguous.  Work items are grouped by column type, then ordered by network
// locality (key bus) so that all consumers of a line's H records / A rows of one
// type run close together and hit in L2.
// One launch per column type (the items are grouped by type): each kernel carries only its
// own code path, so the instruction cache holds it and its registers are its own.
template <bool STRUCT, int TYPE>
__global__ void __launch_bounds__(kMB) k_opf_assemble(OpfKktTab t, In in, int32_t item0,
                                                      int32_t n_items, double* __restrict__ M,
                                                      int32_t* __restrict__ rows,
                                                      int32_t* __restrict__ bad) {
  const int64_t w = ((int64_t)blockIdx.x * kMB + threadIdx.x) >> 5;
  const int32_t lane = threadIdx.x & 31;
  const int64_t it = w / t.tchunks;
  if (it >= n_items) return;
  const int32_t tt = (int32_t)(w - it * t.tchunks) * 32 + lane;
  if (tt >= t.T) return;
  const int32_t e = __ldg(t.items + item0 + it) & 0x0fffffff;
  const int32_t c = lv(t, TYPE, e, tt);
  Out<STRUCT> o{M, rows, __ldg(t.colptr + c)};
  if constexpr (TYPE == C_PG) col_gen<STRUCT, false>(t, in, e, tt, o);
  else if constexpr (TYPE == C_QG) col_gen<STRUCT, true>(t, in, e, tt, o);
  else if constexpr (TYPE == C_P) col_flow<STRUCT, false>(t, in, e, tt, o);
  else if constexpr (TYPE == C_Q) col_flow<STRUCT, true>(t, in, e, tt, o);
  else if constexpr (TYPE == C_V) col_v<STRUCT>(t, in, e, tt, o);
  else col_th<STRUCT>(t, in, e, tt, o);
  if (STRUCT && o.base + o.j != __ldg(t.colptr + c + 1)) atomicOr(bad, 1);
}

template <bool STRUCT>
static void launch_assemble(const OpfKktTab& t, const int32_t* type_lo, const In& in, double* M,
                            int32_t* rows, int32_t* bad, cudaStream_t s) {
  auto go = [&](auto type_tag) {
    constexpr int TY = decltype(type_tag)::value;
    const int32_t n = type_lo[TY + 1] - type_lo[TY];
    if (n <= 0) return;
    const int64_t warps = (int64_t)n * t.tchunks;
    const unsigned blocks = (unsigned)((warps * 32 + kMB - 1) / kMB);
    static const char* names[C_TYPES] = {"k_opf_assemble<pg>", "k_opf_assemble<qg>",
                                         "k_opf_assemble<p>", "k_opf_assemble<q>",
                                         "k_opf_assemble<v>", "k_opf_assemble<th>"};
    KTimer kt(names[TY], s);
    k_opf_assemble<STRUCT, TY><<<blocks, kMB, 0, s>>>(t, in, type_lo[TY], n, M, rows, bad);
    count_launch();
  };
  go(std::integral_constant<int, C_PG>{});
  go(std::integral_constant<int, C_QG>{});
  go(std::integral_constant<int, C_P>{});
  go(std::integral_constant<int, C_Q>{});
  go(std::integral_constant<int, C_V>{});
  go(std::integral_constant<int, C_TH>{});
}

static int64_t assemble_blocks(const OpfKktTab& t) {
  const int64_t warps = (int64_t)t.n_items * t.tchunks;
  return (warps * 32 + kMB - 1) / kMB;
}

// ------------------------------------------------------------ set_jacobian
// One thread per A row; rows are entity-major with t fastest, so both the J
// records and the A rows of a warp are contiguous.  A = 0 (+) J (scatter_values).
__global__ void __launch_bounds__(256) k_opf_set_jac(OpfKktTab t, int32_t m, const double* __restrict__ J,
                                                     double* __restrict__ A) {
  const int64_t r64 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r64 >= m) return;
  const int32_t r = (int32_t)r64, T = t.T;
  const int32_t rp = __ldg(t.rowptr + r);
  if (r < t.flow_p0) {  // balance rows: free generators then incident flows
    const bool Q = r >= t.bal_q0;
    const int32_t rr = r - (Q ? t.bal_q0 : t.bal_p0);
    const int32_t b = rr / T, tt = rr - b * T;
    const int32_t* pos = Q ? t.qpos : t.ppos;
    const int64_t joi = t.jo[Q ? K_BAL_Q_INJ : K_BAL_P_INJ];
    const int64_t jof = t.jo[Q ? K_BAL_Q_FLOW : K_BAL_P_FLOW];
    const int32_t g0 = __ldg(t.bg_ptr + b), g1 = __ldg(t.bg_ptr + b + 1);
    for (int32_t i = g0; i < g1; ++i) {
      const int32_t g = __ldg(t.bg + i);
      const int p = __ldg(pos + g);
      if (p >= 0) A[rp + p] = 0.0 + J[joi + (int64_t)g * T + tt];
    }
    const int nf = __ldg((Q ? t.ngq : t.ngp) + b);
    const int32_t b0 = __ldg(t.bl_ptr + b), b1 = __ldg(t.bl_ptr + b + 1);
    for (int32_t i = b0; i < b1; ++i) {
      const int32_t e = __ldg(t.bl + i), l = e >> 1, fr = e & 1;
      A[rp + nf + (i - b0)] = 0.0 + J[jof + 2 * ((int64_t)l * T + tt) + fr];
    }
  } else if (r < t.therm0) {  // flow definitions
    const bool Q = r >= t.flow_q0;
    const int32_t rr = r - (Q ? t.flow_q0 : t.flow_p0);
    const int32_t l = rr / T;
    const double* src = J + t.jo[Q ? K_FLOW_Q : K_FLOW_P] + 5 * (int64_t)rr;
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      const int p = __ldg(t.fpos + 5 * l + f);
      if (p >= 0) A[rp + p] = 0.0 + src[f];
    }
  } else if (r < t.ang0) {  // thermal [p, q]
    const double* src = J + t.jo[K_THERMAL] + 2 * (int64_t)(r - t.therm0);
    A[rp] = 0.0 + src[0];
    A[rp + 1] = 0.0 + src[1];
  } else if (r < t.ramp0) {  // angle [th_f, th_t]
    const int32_t rr = r - t.ang0, l = rr / T;
    const double* src = J + t.jo[K_ANGLE] + 2 * (int64_t)rr;
    const int pf = __ldg(t.apos + 2 * l), pt = __ldg(t.apos + 2 * l + 1);
    if (pf >= 0) A[rp + pf] = 0.0 + src[0];
    if (pt >= 0) A[rp + pt] = 0.0 + src[1];
  } else {  // ramp [pg_t, pg_{t-1}] -> CSR order [pg_{t-1}, pg_t]
    const int32_t len = __ldg(t.rowptr + r + 1) - rp;
    if (len == 2) {
      const double* src = J + t.jo[K_RAMP] + 2 * (int64_t)(r - t.ramp0);
      A[rp] = 0.0 + src[1];
      A[rp + 1] = 0.0 + src[0];
    }
  }
}

__global__ void k_count_diff(const int32_t* a, const int32_t* b, int64_t n, int32_t* diff) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && a[i] != b[i]) atomicAdd(diff, 1);
}
void count_diff(const int32_t* a, const int32_t* b, int64_t n, int32_t* diff, cudaStream_t s) {
  if (n <= 0) return;
  k_count_diff<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, n, diff);
  count_launch();
}

// --------------------------------------------------------------- host setup
template <class T>
static void up(DBuf<T>& b, const std::vector<T>& v, cudaStream_t s) {
  b.upload(v.data(), v.size(), s);
  if (v.empty()) b.alloc(1);
}

bool opf_kkt_prepare(gn_kkt* K) {
  gn_ctx* c = K->ctx;
  const OpfDims& d = c->d;
  cudaStream_t s = K->stream;
  auto* X = new OpfKkt();
  K->opf = X;
  // Self-loop lines (from == to) fold two fields of a record onto one variable; the
  // topology-walking kernels assume two distinct terminals, so such a network keeps the
  // generic assembly (any COO structure; bit-identical to the reference as well) and has no
  // fused path.
  for (int32_t l = 0; l < d.L; ++l)
    if (c->line_from[l] == c->line_to[l]) return false;
  OpfKktTab& t = X->t;
  t.T = d.T; t.N = d.N; t.L = d.L; t.G = d.G;
  t.bal_p0 = d.bal_p0; t.bal_q0 = d.bal_q0; t.flow_p0 = d.flow_p0; t.flow_q0 = d.flow_q0;
  t.therm0 = d.therm0; t.ang0 = d.ang0; t.ramp0 = d.ramp0;
  for (int q = 0; q < K_COUNT; ++q) { t.ho[q] = d.hess_off[q]; t.jo[q] = d.jac_off[q]; }
  const int32_t N = d.N, L = d.L, G = d.G;
  // free entities (lifted.hpp:140-147 on the per-entity boxes)
  std::vector<uint8_t> fixed = c->fixed_ent;
  std::vector<int32_t> lent(fixed.size(), -1);
  int32_t rank = 0;
  for (size_t e = 0; e < fixed.size(); ++e) lent[e] = fixed[e] ? -1 : rank++;
  const int32_t offs[C_TYPES + 1] = {0, G, 2 * G, 2 * G + L, 2 * G + 2 * L, 2 * G + 2 * L + N,
                                     2 * G + 2 * L + 2 * N};
  // work items in network-locality order: (key bus, type, entity)
  std::vector<std::pair<int64_t, int32_t>> order;
  int64_t nfree_ent = 0;
  for (int ty = 0; ty < C_TYPES; ++ty)
    for (int32_t e = 0; e < offs[ty + 1] - offs[ty]; ++e) {
      if (fixed[offs[ty] + e]) continue;
      ++nfree_ent;
      int32_t key;
      if (ty == C_PG || ty == C_QG) key = c->gen_bus[e];
      else if (ty == C_P || ty == C_Q) key = std::min(c->line_from[e], c->line_to[e]);
      else key = e;
      // grouped by column type first (neighbouring warps run the same code path: the
      // kernel's per-type paths no longer thrash the instruction cache), then by
      // network locality (key bus) within a type
      order.push_back({((int64_t)ty << 59) | ((int64_t)key << 28) | e, (ty << 28) | e});
    }
  std::sort(order.begin(), order.end());
  std::vector<int32_t> items;
  items.reserve(order.size());
  for (auto& pr : order) items.push_back(pr.second);
  t.n_items = static_cast<int32_t>(items.size());
  for (int ty = 0; ty <= C_TYPES; ++ty) X->type_lo[ty] = 0;
  for (auto& pr : order) ++X->type_lo[(pr.second >> 28) + 1];
  for (int ty = 0; ty < C_TYPES; ++ty) X->type_lo[ty + 1] += X->type_lo[ty];
  t.tchunks = (d.T + 31) / 32;
  auto vfree = [&](int32_t n) { return !fixed[offs[C_V] + n]; };
  auto tfree = [&](int32_t n) { return !fixed[offs[C_TH] + n]; };
  // per-bus incidence (ascending l), generator ranks
  std::vector<std::vector<int32_t>> inc(N), gens(N);
  for (int32_t l = 0; l < L; ++l) {
    inc[c->line_to[l]].push_back(l << 1);
    inc[c->line_from[l]].push_back((l << 1) | 1);
  }
  for (auto& v : inc) std::sort(v.begin(), v.end());
  for (int32_t g = 0; g < G; ++g) gens[c->gen_bus[g]].push_back(g);
  std::vector<int32_t> lidx_to(L), lidx_from(L), bl_ptr(N + 1, 0), bl, bg_ptr(N + 1, 0), bg;
  std::vector<int32_t> ngp(N, 0), ngq(N, 0), ppos(G, -1), qpos(G, -1), g_ramp(G, -1);
  for (int32_t n = 0; n < N; ++n) {
    for (size_t i = 0; i < inc[n].size(); ++i) {
      const int32_t l = inc[n][i] >> 1;
      if (inc[n][i] & 1) lidx_from[l] = static_cast<int32_t>(i); else lidx_to[l] = static_cast<int32_t>(i);
      bl.push_back(inc[n][i]);
    }
    bl_ptr[n + 1] = static_cast<int32_t>(bl.size());
    for (int32_t g : gens[n]) {
      bg.push_back(g);
      if (!fixed[offs[C_PG] + g]) ppos[g] = ngp[n]++;
      if (!fixed[offs[C_QG] + g]) qpos[g] = ngq[n]++;
    }
    bg_ptr[n + 1] = static_cast<int32_t>(bg.size());
  }
  for (int32_t k = 0; k < d.GR; ++k) g_ramp[c->ramp_gens[k]] = k;
  std::vector<int32_t> l_therm(L, -1);
  for (int32_t k = 0; k < d.LT; ++k) l_therm[c->thermal_lines[k]] = k;
  // neighbour-grouped incidence (other bus, l)
  std::vector<int32_t> nb_ptr(N + 1, 0), nb, nb_inc;
  int32_t maxdeg = 0;
  for (int32_t n = 0; n < N; ++n) {
    std::vector<std::pair<std::pair<int32_t, int32_t>, int32_t>> v;
    for (size_t i = 0; i < inc[n].size(); ++i) {
      const int32_t e = inc[n][i], l = e >> 1;
      v.push_back({{(e & 1) ? c->line_to[l] : c->line_from[l], e}, static_cast<int32_t>(i)});
    }
    std::sort(v.begin(), v.end());
    for (auto& pr : v) {
      nb.push_back(pr.first.second);
      nb_inc.push_back(pr.second);
    }
    nb_ptr[n + 1] = static_cast<int32_t>(nb.size());
    maxdeg = std::max(maxdeg, static_cast<int32_t>(inc[n].size()));
  }
  t.maxdeg = maxdeg;
  // slot programs of the fused bus-column kernel (gn_opf_fused_bus.cu): rows of
  // v(n) then th(n) in CSC order, each with the lane mask of its lines
  std::vector<int32_t> bprog_ptr(N + 1, 0);
  std::vector<unsigned long long> bprog;
  if (maxdeg <= 32) {
    auto slot = [&](uint32_t mask, int type, int32_t ent) {
      bprog.push_back((static_cast<unsigned long long>(ent) << 35) |
                      (static_cast<unsigned long long>(type) << 32) | mask);
    };
    for (int32_t n = 0; n < N; ++n) {
      const int32_t deg = static_cast<int32_t>(inc[n].size());
      const uint32_t all = deg >= 32 ? 0xffffffffu : ((1u << deg) - 1u);
      // neighbour groups (ascending other bus): lane mask of the group's lines
      std::vector<std::pair<int32_t, uint32_t>> groups;
      for (int32_t u = nb_ptr[n]; u < nb_ptr[n + 1]; ++u) {
        const int32_t e = nb[u], l = e >> 1;
        const int32_t ob = (e & 1) ? c->line_to[l] : c->line_from[l];
        if (groups.empty() || groups.back().first != ob) groups.push_back({ob, 0u});
        groups.back().second |= 1u << nb_inc[u];
      }
      const bool vfree_n = !fixed[offs[C_V] + n], tfree_n = !fixed[offs[C_TH] + n];
      if (vfree_n) {
        slot(all, 0, n);
        for (auto& gp : groups)
          if (gp.first > n && !fixed[offs[C_V] + gp.first]) slot(gp.second, 1, gp.first);
        bool self = false;
        for (size_t k = 0; k <= groups.size(); ++k) {
          const int32_t ob = k < groups.size() ? groups[k].first : 0x7fffffff;
          if (!self && n < ob) {
            self = true;
            if (tfree_n && deg > 0) slot(all, 2, n);  // no (th(n), v(n)) without lines
          }
          if (k < groups.size() && !fixed[offs[C_TH] + ob]) slot(groups[k].second, 3, ob);
        }
      }
      if (tfree_n) {
        slot(all, 4, n);
        for (auto& gp : groups)
          if (gp.first > n && !fixed[offs[C_TH] + gp.first]) slot(gp.second, 5, gp.first);
      }
      bprog_ptr[n + 1] = static_cast<int32_t>(bprog.size());
    }
  }
  t.pg0 = d.pg0; t.qg0 = d.qg0; t.p0 = d.p0; t.q0 = d.q0; t.v0 = d.v0; t.th0 = d.th0;
  t.s_lo = d.s_lo; t.R = d.R; t.prev = d.prev; t.next = d.next;
  t.grid_cap = grid_cap_default();
  t.lg = c->lg.p; t.lb = c->lb.p; t.c2 = c->c2.p; t.th_line = c->th_line.p;
  // flow-row / angle-row positions
  std::vector<int8_t> fpos(5 * static_cast<size_t>(L)), apos(2 * static_cast<size_t>(L));
  for (int32_t l = 0; l < L; ++l) {
    const int32_t f = c->line_from[l], to = c->line_to[l];
    // candidate columns in CSR order: p, v(min), v(max), th(min), th(max)
    int8_t pos = 0;
    fpos[5 * l] = pos++;
    const int32_t lo = std::min(f, to), hi = std::max(f, to);
    int8_t pv_lo = vfree(lo) ? pos++ : -1, pv_hi = vfree(hi) ? pos++ : -1;
    int8_t pt_lo = tfree(lo) ? pos++ : -1, pt_hi = tfree(hi) ? pos++ : -1;
    fpos[5 * l + 1] = f == lo ? pv_lo : pv_hi;
    fpos[5 * l + 2] = to == lo ? pv_lo : pv_hi;
    fpos[5 * l + 3] = f == lo ? pt_lo : pt_hi;
    fpos[5 * l + 4] = to == lo ? pt_lo : pt_hi;
    int8_t a = 0;
    int8_t a_lo = tfree(lo) ? a++ : -1, a_hi = tfree(hi) ? a++ : -1;
    apos[2 * l] = f == lo ? a_lo : a_hi;
    apos[2 * l + 1] = to == lo ? a_lo : a_hi;
  }
  // line neighbours l' > l sharing a bus; bits: 1 = shares min(f,to), 2 = shares max
  std::vector<int32_t> lnb_ptr(L + 1, 0), lnb, lnbx;
  for (int32_t l = 0; l < L; ++l) {
    const int32_t f = c->line_from[l], to = c->line_to[l];
    const int32_t lo = std::min(f, to), hi = std::max(f, to);
    std::vector<std::pair<int32_t, int32_t>> v;
    for (int side = 0; side < 2; ++side) {
      const int32_t b = side ? hi : lo;
      for (int32_t e : inc[b]) {
        const int32_t l2 = e >> 1;
        if (l2 > l) v.push_back({l2, side ? 2 : 1});
      }
    }
    std::sort(v.begin(), v.end());
    for (size_t i = 0; i < v.size();) {
      int32_t bits = 0, l2 = v[i].first;
      while (i < v.size() && v[i].first == l2) bits |= v[i++].second;
      lnb.push_back((l2 << 2) | bits);
      // fused line kernel: + the balance-row signs of l2 at the shared buses
      const int32_t to2 = c->line_to[l2];
      lnbx.push_back((l2 << 4) | bits | (lo == to2 ? 4 : 0) | (hi == to2 ? 8 : 0));
    }
    lnb_ptr[l + 1] = static_cast<int32_t>(lnb.size());
  }
  // per-line descriptors of the fused line kernel (one level of independent loads)
  std::vector<int4> ldesc0(L), ldesc1(L);
  for (int32_t l = 0; l < L; ++l) {
    const int32_t f = c->line_from[l], to = c->line_to[l];
    const int32_t lo = std::min(f, to), hi = std::max(f, to);
    const int32_t flags = (vfree(lo) ? 1 : 0) | (vfree(hi) ? 2 : 0) | (tfree(lo) ? 4 : 0) |
                          (tfree(hi) ? 8 : 0) | (lo == to ? 16 : 0) | (hi == to ? 32 : 0);
    ldesc0[l] = make_int4(f, to, l_therm[l], flags);
    ldesc1[l] = make_int4(lnb_ptr[l], lnb_ptr[l + 1], lent[offs[C_P] + l], lent[offs[C_Q] + l]);
  }
  up(X->lent, lent, s); up(X->items, items, s);
  up(X->lf, c->line_from, s); up(X->lt, c->line_to, s); up(X->l_therm, l_therm, s);
  up(X->fpos, fpos, s); up(X->apos, apos, s); up(X->lidx_to, lidx_to, s); up(X->lidx_from, lidx_from, s);
  up(X->gbus, c->gen_bus, s); up(X->ppos, ppos, s); up(X->qpos, qpos, s); up(X->g_ramp, g_ramp, s);
  up(X->ngp, ngp, s); up(X->ngq, ngq, s); up(X->bl_ptr, bl_ptr, s); up(X->bl, bl, s);
  up(X->bg_ptr, bg_ptr, s); up(X->bg, bg, s); up(X->nb_ptr, nb_ptr, s); up(X->nb, nb, s); up(X->nb_inc, nb_inc, s);
  up(X->lnb_ptr, lnb_ptr, s); up(X->lnb, lnb, s); up(X->lnbx, lnbx, s);
  up(X->ldesc0, ldesc0, s); up(X->ldesc1, ldesc1, s);
  up(X->bprog_ptr, bprog_ptr, s); up(X->bprog, bprog, s);
  {  // bus-column kernel: per incident line (bl order) its (l<<1|is_from, other bus) and (G, B);
     // per degree class the bus descriptors (n, bl begin, deg | program length << 8,
     // program begin) + (lifted v rank, lifted th rank)
    std::vector<int2> blx(bl.size());
    std::vector<double2> blgb(bl.size());
    std::vector<double> lg_h(L), lb_h(L);
    if (L > 0) {
      GN_CK(cudaMemcpyAsync(lg_h.data(), c->lg.p, sizeof(double) * L, cudaMemcpyDeviceToHost, s));
      GN_CK(cudaMemcpyAsync(lb_h.data(), c->lb.p, sizeof(double) * L, cudaMemcpyDeviceToHost, s));
      GN_CK(cudaStreamSynchronize(s));
    }
    for (size_t i = 0; i < bl.size(); ++i) {
      const int32_t e = bl[i], l = e >> 1;
      blx[i] = make_int2(e, (e & 1) ? c->line_to[l] : c->line_from[l]);
      blgb[i] = make_double2(lg_h[l], lb_h[l]);
    }
    up(X->blx, blx, s);
    up(X->blgb, blgb, s);
    // Register-resident classes (buses of exactly DEG = 1..6 lines, no parallel lines):
    // per incidence the in-column offsets of its neighbour slots, read off the slot
    // program: (v(o), v(n)) | (th(o), v(n)) << 8 | (th(o), th(n)) << 16, 0xff = absent.
    std::vector<int32_t> bpos(bl.size(), 0xffffff);
    std::vector<int4> cls[kBusClasses];
    // M column starts/lengths of v(n), th(n): a column's slots are the same for every
    // period, so column (k, t) starts at colptr[k*T] + t * len(k) -- held in the bus
    // descriptor, no colptr lookup on the kernels' critical path
    std::vector<int32_t> cp(static_cast<size_t>(K->n) + 1);
    GN_CK(cudaMemcpyAsync(cp.data(), K->M.ptr.p, sizeof(int32_t) * cp.size(), cudaMemcpyDeviceToHost, s));
    GN_CK(cudaStreamSynchronize(s));
    {  // row / column starts at t = 0 of the fused kernels' entities (same reason)
      std::vector<int32_t> rp(static_cast<size_t>(K->m) + 1);
      GN_CK(cudaMemcpyAsync(rp.data(), K->A.ptr.p, sizeof(int32_t) * rp.size(),
                            cudaMemcpyDeviceToHost, s));
      GN_CK(cudaStreamSynchronize(s));
      const int64_t TT = d.T;
      std::vector<int32_t> rbase(2 * static_cast<size_t>(N) + 3 * static_cast<size_t>(L) + d.LT);
      for (int32_t b = 0; b < N; ++b) {
        rbase[b] = rp[d.bal_p0 + b * TT];
        rbase[N + b] = rp[d.bal_q0 + b * TT];
      }
      for (int32_t l = 0; l < L; ++l) {
        rbase[2 * N + l] = rp[d.flow_p0 + l * TT];
        rbase[2 * N + L + l] = rp[d.flow_q0 + l * TT];
        rbase[2 * N + 2 * L + d.LT + l] = rp[d.ang0 + l * TT];
      }
      for (int32_t k = 0; k < d.LT; ++k) rbase[2 * N + 2 * L + k] = rp[d.therm0 + k * TT];
      std::vector<int2> lcb(L);
      for (int32_t l = 0; l < L; ++l) {
        const int32_t kp = lent[offs[C_P] + l], kq = lent[offs[C_Q] + l];
        lcb[l] = make_int2(kp >= 0 ? cp[kp * TT] : 0, kq >= 0 ? cp[kq * TT] : 0);
      }
      up(X->rbase, rbase, s);
      up(X->lcb, lcb, s);
    }
    auto colspan = [&](int32_t k, int32_t& base, int32_t& len) {
      base = len = 0;
      if (k < 0) return;
      const int64_t c = static_cast<int64_t>(k) * d.T;
      base = cp[c];
      len = cp[c + 1] - cp[c];
    };
    for (int32_t n = 0; n < N; ++n) {
      const int32_t deg = bl_ptr[n + 1] - bl_ptr[n];
      const int32_t np = bprog_ptr[n + 1] - bprog_ptr[n];
      bool simple = deg >= 1 && deg <= kBusRegMax;
      int32_t jv = 0, jt = 0, boff_n = -1;
      for (int32_t q = bprog_ptr[n]; q < bprog_ptr[n + 1]; ++q) {
        const unsigned long long code = bprog[q];
        const uint32_t mask = static_cast<uint32_t>(code);
        const int type = static_cast<int>((code >> 32) & 7);
        const int32_t j = type < 4 ? jv++ : jt++;
        if (type == 2) boff_n = j;
        if (type == 1 || type == 3 || type == 5) {
          if (mask & (mask - 1)) {  // parallel lines: generic kernel
            simple = false;
            continue;
          }
          const int i = __builtin_ctz(mask), sh = type == 1 ? 0 : (type == 3 ? 8 : 16);
          int32_t& b = bpos[bl_ptr[n] + i];
          b = (b & ~(0xff << sh)) | (j << sh);
        }
      }
      if (simple) {
        cls[deg - 1].push_back(make_int4(n, bl_ptr[n], deg, boff_n));
      } else {
        cls[(deg <= 8 && !GN_BUS3_MERGE) ? kBusClasses - 2 : kBusClasses - 1].push_back(
            make_int4(n, bl_ptr[n], deg | (np << 8), bprog_ptr[n]));
      }
      auto& v = simple ? cls[deg - 1]
                       : cls[(deg <= 8 && !GN_BUS3_MERGE) ? kBusClasses - 2 : kBusClasses - 1];
      const int32_t kv = lent[offs[C_V] + n], kt = lent[offs[C_TH] + n];
      int32_t bv, lv, bt, lt;
      colspan(kv, bv, lv);
      colspan(kt, bt, lt);
      v.push_back(make_int4(kv, kt, 0, 0));
      v.push_back(make_int4(bv, lv, bt, lt));
      if (simple) {  // register classes: the incident lines inline (one level of loads)
        for (int32_t i = 0; i < deg; ++i) {
          const int2 e = blx[bl_ptr[n] + i];
          v.push_back(make_int4(e.x, e.y, bpos[bl_ptr[n] + i], 0));
        }
        for (int32_t i = 0; i < deg; ++i) {
          int4 gbits;
          std::memcpy(&gbits, &blgb[bl_ptr[n] + i], sizeof gbits);  // (G, B) as 16 bytes
          v.push_back(gbits);
        }
      }
    }
    up(X->bpos, bpos, s);
    for (int k = 0; k < kBusClasses; ++k) {
      up(X->bus_cls[k], cls[k], s);
      if (cls[k].empty()) X->bus_cls[k].alloc(kBusDesc);
      X->n_bus_cls[k] = static_cast<int32_t>(cls[k].size() / bus_desc_stride(k));
    }
    int32_t md = 0;
    for (size_t i = 0; i < cls[kBusClasses - 1].size(); i += kBusDesc)
      md = std::max(md, cls[kBusClasses - 1][i].z & 255);
    X->maxdeg_rest = md;
  }
  t.lent = X->lent.p; t.items = X->items.p; t.lf = X->lf.p; t.lt = X->lt.p; t.l_therm = X->l_therm.p;
  t.fpos = X->fpos.p; t.apos = X->apos.p; t.lidx_to = X->lidx_to.p; t.lidx_from = X->lidx_from.p;
  t.gbus = X->gbus.p; t.ppos = X->ppos.p; t.qpos = X->qpos.p; t.g_ramp = X->g_ramp.p;
  t.ngp = X->ngp.p; t.ngq = X->ngq.p; t.bl_ptr = X->bl_ptr.p; t.bl = X->bl.p;
  t.bg_ptr = X->bg_ptr.p; t.bg = X->bg.p; t.nb_ptr = X->nb_ptr.p; t.nb = X->nb.p; t.nb_inc = X->nb_inc.p;
  t.lnb_ptr = X->lnb_ptr.p; t.lnb = X->lnb.p; t.lnbx = X->lnbx.p;
  t.blx = X->blx.p; t.blgb = X->blgb.p; t.bpos = X->bpos.p;
  t.rbase = X->rbase.p; t.lcb = X->lcb.p;
  t.ldesc0 = X->ldesc0.p; t.ldesc1 = X->ldesc1.p;
  t.bprog_ptr = X->bprog_ptr.p; t.bprog = X->bprog.p;
  t.rowptr = K->A.ptr.p; t.colptr = K->M.ptr.p;
  GN_CK(cudaStreamSynchronize(s));

  // Verify the enumeration against the generic CSC (row index of every slot).
  const int64_t blocks = assemble_blocks(t);
  t.n_owned = static_cast<int32_t>(nfree_ent * d.T);
  const bool shard = d.prev || d.next;  // the contract kernels assume a whole horizon
  bool ok = !shard && nfree_ent * d.T == K->n;
  if (ok && blocks > 0) {
    DBuf<int32_t> rows, bad;
    rows.alloc(static_cast<size_t>(K->mnnz) + 1);
    bad.alloc(1);
    GN_CK(cudaMemsetAsync(bad.p, 0, 4, s));
    In in{};
    launch_assemble<true>(t, X->type_lo, in, nullptr, rows.p, bad.p, s);
    GN_CK(cudaGetLastError());
    int32_t hb = 0;
    GN_CK(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
    GN_CK(cudaStreamSynchronize(s));
    ok = hb == 0;
    if (ok) {  // compare row indices with the generic build
      DBuf<int32_t> diff;
      diff.alloc(1);
      GN_CK(cudaMemsetAsync(diff.p, 0, 4, s));
      count_diff(rows.p, K->M.idx.p, K->mnnz, diff.p, s);
      GN_CK(cudaMemcpyAsync(&hb, diff.p, 4, cudaMemcpyDeviceToHost, s));
      GN_CK(cudaStreamSynchronize(s));
      ok = hb == 0;
    }
  }
  X->ready = ok;
  X->fused_ready = (nfree_ent * d.T + (d.next ? d.GR : 0) == K->n) && opf_fused_verify(K);
  return ok;
}

bool opf_kkt_ready(const gn_kkt* K) { return K->opf && K->opf->ready; }

void opf_set_grid_cap(gn_kkt* K, int ctas_per_sm) {
  if (K->opf) K->opf->t.grid_cap = ctas_per_sm;
}

void opf_kkt_free(gn_kkt* K) {
  delete K->opf;
  K->opf = nullptr;
}

void opf_set_jacobian(gn_kkt* K, const double* Jfull) {
  const OpfKktTab& t = K->opf->t;
  if (K->m <= 0) return;
  KTimer kt("k_opf_set_jac", K->stream);
  k_opf_set_jac<<<(unsigned)((K->m + 255) / 256), 256, 0, K->stream>>>(t, K->m, Jfull, K->avals.p);
  count_launch();
  GN_CK(cudaGetLastError());
}

void opf_assemble(gn_kkt* K, const double* Hfull, const double* sx, const double* ss, double dw,
                  double dc) {
  const OpfKktTab& t = K->opf->t;
  const int64_t blocks = assemble_blocks(t);
  if (blocks <= 0) return;
  launch_dvec(K, ss, dw, dc);
  In in{Hfull, K->avals.p, sx, K->dvals.p, dw};
  launch_assemble<false>(t, K->opf->type_lo, in, K->mvals.p, nullptr, nullptr, K->stream);
  GN_CK(cudaGetLastError());
}

}  // namespace gnb
