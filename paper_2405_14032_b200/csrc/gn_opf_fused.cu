// Fused condensed-KKT kernels: A and M straight from the primal point x.
//
// CondensedKkt::assemble(H, Sx, Ss, dw, dc) reads the Hessian the callback just
// wrote and the CSR Jacobian values; on the device both are pure functions of
// (x, row weights, obj weight).  These kernels recompute every contributing H
// entry and A entry in registers with the *same* device expressions the
// callbacks use (gn_opf_math.cuh, -fmad=false), so
//     assemble_fused(x, w, ow, ...) == assemble(eval_hess(x, w, ow), set_jacobian(eval_jac(x)), ...)
// bit for bit, while the ~2 GB/unit of H and A read-back disappears from HBM.
// Contributors are added in the reference order (condensed.hpp:118-134,
// SURVEY A.5); contributors that are identically +-0 (structural zeros of the
// Hessian) are skipped, which cannot change the sum because an accumulator
// that starts at +0.0 never becomes -0.0.
//
// Work decomposition: one warp per (bus n, 32 consecutive periods), lane = period.
// The warp owns the columns v(n), th(n), p(l)/q(l) of the lines whose smaller
// terminal is n, and pg(g)/qg(g) of the generators at n.  Each incident line's
// trigonometric state is computed once per lane and kept in shared memory.
#include <cstdlib>

#include "gn_opf_kkt.cuh"
#include "gn_opf_math.cuh"
#include "gn_span.cuh"

namespace gnb {



template <bool STRUCT>
struct FOut {
  double* M;
  int32_t* rows;
  int64_t base;
  int j;
  __device__ __forceinline__ void put(double v, int32_t row) {
    if constexpr (STRUCT) rows[base + j] = row; else M[base + j] = v;
    ++j;
  }
};

__device__ __forceinline__ int32_t f_lent(const OpfKktTab& t, int32_t off, int32_t e) {
  return __ldg(t.lent + off + e);
}

struct Ctx {
  const OpfKktTab& t;
  const FIn& in;
  int32_t n, tt, T;
  int32_t b0, deg;
  double* S;  // unused by the line/generator kernels
  int lane;
  const double* dv;  // d_r per row (k_fz_dvec)
  int32_t off_pg, off_qg, off_p, off_q, off_v, off_th;

  __device__ int32_t inc(int i) const { return __ldg(t.bl + b0 + i); }
  __device__ LineState st(int i) const {
    const double* q = S + (i * 6) * 32 + lane;
    LineState s;
    s.vf = q[0];
    s.vt = q[32];
    s.vfvt = s.vf * s.vt;
    s.Cs = q[64];
    s.Sn = q[96];
    s.cs = q[128];
    s.sn = q[160];
    return s;
  }
  __device__ double d(int32_t row) const { return dval(t, dv, row); }
  __device__ double wt(int32_t row) const { return in.w[row]; }
  __device__ int32_t col(int32_t off, int32_t e) const {
    const int32_t k = f_lent(t, off, e);
    return k < 0 ? -1 : k * T + tt;
  }
};

// pg(g) and qg(g) columns of generator g at period c.tt (thread per (g, t)).
template <bool STRUCT>
__device__ void fz_gen_cols(const Ctx& c, int32_t gsel, double* M, int32_t* rows, int32_t* bad) {
  const OpfKktTab& t = c.t;
  const FIn& in = c.in;
  const int32_t T = c.T, tt = c.tt;
  const int32_t n = __ldg(t.gbus + gsel);
  const int32_t b0 = __ldg(t.bl_ptr + n), deg = __ldg(t.bl_ptr + n + 1) - b0;
  auto check = [&](const FOut<STRUCT>& o, int32_t cc) {
    if (STRUCT && o.base + o.j != __ldg(t.colptr + cc + 1)) atomicOr(bad, 1);
  };
  const int32_t g0 = __ldg(t.bg_ptr + n), g1 = __ldg(t.bg_ptr + n + 1);
  {
    const int32_t g = gsel;
#pragma unroll
    for (int Q = 0; Q < 2; ++Q) {
      const int32_t cc = c.col(Q ? c.off_qg : c.off_pg, g);
      if (cc < 0) continue;
      FOut<STRUCT> o{M, rows, __ldg(t.colptr + cc), 0};
      const int32_t rb = (Q ? t.bal_q0 : t.bal_p0) + n * T + tt;
      const int32_t kr = Q ? -1 : __ldg(t.g_ramp + g);
      // ramp row of step s = s_lo .. s_lo + R - 1: row (k, s) couples pg(s-1), pg(s)
      const bool lo_ok = kr >= 0 && tt >= t.s_lo;              // row (k, tt) exists
      const bool hi_ok = kr >= 0 && tt + 1 <= t.s_lo + t.R - 1;  // row (k, tt+1) exists
      const bool ghost = hi_ok && tt + 1 == T;  // its pg(tt+1) is the next rank's (ghost)
      const int32_t rr = t.ramp0 + (kr >= 0 ? kr : 0) * t.R - t.s_lo;  // + s = row of step s
      {
        double acc = 0.0;
        if constexpr (!STRUCT) {
          if (!Q) acc += h_cost(in.ow, __ldg(t.c2 + g));
          acc += pair_term(c.d(rb), 1.0, 1.0);
          if (lo_ok) acc += pair_term(c.d(rr + tt), 1.0, 1.0);
          if (hi_ok) acc += pair_term(c.d(rr + tt + 1), -1.0, -1.0);
          acc += in.dw + in.sx[cc];
        }
        o.put(acc, cc);
      }
      if (hi_ok && !ghost) {  // (pg(g,t+1), pg(g,t))
        double acc = 0.0;
        if constexpr (!STRUCT) acc += pair_term(c.d(rr + tt + 1), 1.0, -1.0);
        o.put(acc, cc + 1);
      }
      for (int32_t gj = g0; gj < g1; ++gj) {
        const int32_t g2 = __ldg(t.bg + gj);
        if (g2 <= g) continue;
        const int32_t c2c = c.col(Q ? c.off_qg : c.off_pg, g2);
        if (c2c < 0) continue;
        double acc = 0.0;
        if constexpr (!STRUCT) acc += pair_term(c.d(rb), 1.0, 1.0);
        o.put(acc, c2c);
      }
      for (int i = 0; i < deg; ++i) {
        const int32_t e = __ldg(t.bl + b0 + i), l = e >> 1;
        double acc = 0.0;
        if constexpr (!STRUCT) acc += pair_term(c.d(rb), (e & 1) ? -1.0 : 1.0, 1.0);
        o.put(acc, c.col(Q ? c.off_q : c.off_p, l));
      }
      if (ghost) {  // (pg_next ghost, pg(g, T-1)): the ghost's lifted index is after every owned column
        double acc = 0.0;
        if constexpr (!STRUCT) acc += pair_term(c.d(rr + tt + 1), 1.0, -1.0);
        o.put(acc, t.n_owned + kr);
      }
      check(o, cc);
    }
  }
}

// d_r for every row (condensed.hpp:111-117), once per assemble call.
// Four rows per thread with 16-byte loads / stores (when sigma_s is 16-byte aligned; the
// d buffer is ours and always is): a pure stream, so wide accesses and more bytes in
// flight per thread are what move it toward the copy bandwidth.
__global__ void __launch_bounds__(256) k_fz_dvec(int32_t m, const double* __restrict__ ss, double dw,
                                                 double dc, double* __restrict__ dv) {
  const int64_t r0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (r0 >= m) return;
  if (r0 + 4 <= m && (reinterpret_cast<uintptr_t>(ss) & 15) == 0) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(ss + r0));
    const double2 b = __ldg(reinterpret_cast<const double2*>(ss + r0 + 2));
    reinterpret_cast<double2*>(dv + r0)[0] = make_double2(dvec(a.x, dw, dc), dvec(a.y, dw, dc));
    reinterpret_cast<double2*>(dv + r0)[1] = make_double2(dvec(b.x, dw, dc), dvec(b.y, dw, dc));
  } else {
    for (int64_t r = r0; r < r0 + 4 && r < m; ++r) dv[r] = dvec(ss[r], dw, dc);
  }
}

// p(l) and q(l) columns of line l, one warp per (l, 32 consecutive periods),
// lane = period.
//
//   rows of p(l): p(l) | p(l') for l' > l sharing a bus | q(l) if thermal | v(lo) v(hi) th(lo) th(hi)
//   rows of q(l): q(l) | q(l') ...                                         | v(lo) v(hi) th(lo) th(hi)
//
// (lo, hi = min / max terminal; v/th rows only where free.)  Every input comes
// from one level of per-line descriptors (independent loads, restrict-qualified
// so none waits behind an M store).  The columns of consecutive periods are
// consecutive in M, so a warp's p (then q) columns form one contiguous span:
// lanes stage their column in shared memory ([slot][lane], conflict-free) and
// the warp writes the span back coalesced.  Direct per-lane writes would make
// every 8-byte store its own L2 sector write (4x the write transactions, and
// partial-sector fills from HBM).
// resident-CTA floors of the launch bounds (register caps); overridable for tuning builds
// (scripts/build_variant.py)
#ifndef GN_FL_GS_MINB
#define GN_FL_GS_MINB 6
#endif
#ifndef GN_SJ_MINB
#define GN_SJ_MINB 6
#endif
#ifndef GN_SJ_GS_MINB
#define GN_SJ_GS_MINB 6
#endif
#ifndef GN_FLW
#define GN_FLW 4
#endif
constexpr int kFLW = GN_FLW;  // warps per CTA
// flow-column kernel: flat (line, period) lanes when T is not a multiple of 32 (no idle lanes:
// 9241 x 48 -12%, a 21-period shard -16%), a warp per (line, 32 periods) otherwise (flat costs
// 2% at 96 periods: prefix sums, per-lane descriptors).  GN_FL_FLAT=0: never flat.
#ifndef GN_FL_FLAT
#define GN_FL_FLAT 1
#endif
#ifndef GN_FLCAP
#define GN_FLCAP 16  // 12: 30k x 96 =, 9241 x 48 +0.5%; 24 (25 KB of staging per CTA): +6-10%
#endif
constexpr int kFLCap = GN_FLCAP;  // staged slots per column (longer columns are written in place)
template <bool STRUCT, bool FLAT = false>
__device__ __forceinline__ void fz_line_body(int64_t vblock, const OpfKktTab& t,
                                             const double* __restrict__ x,
                                             const double* __restrict__ w,
                                             const double* __restrict__ sx, double dw,
                                             const double* __restrict__ dv,
                                             double* __restrict__ M,
                                             int32_t* __restrict__ rows,
                                             int32_t* __restrict__ bad) {
  __shared__ double stg_all[STRUCT ? 1 : kFLW * kFLCap * 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t T = t.T;
  const int64_t wg = vblock * kFLW + warp;
  constexpr bool flat = !STRUCT && FLAT;
  int32_t l, tt, c0 = 0, nt = 0;
  bool valid;
  if constexpr (flat) {  // lane = item 32 wg + lane of the flat (line, period) order
    const int64_t nitems = (int64_t)t.L * T, item = wg * 32 + lane;
    if (wg * 32 >= nitems) return;  // warp-uniform
    valid = item < nitems;
    const int64_t it = valid ? item : nitems - 1;
    l = (int32_t)(it / T);
    tt = (int32_t)(it - (int64_t)l * T);
  } else {
    l = (int32_t)(wg / t.tchunks);
    if (l >= t.L) return;  // warp-uniform
    c0 = (int32_t)(wg - (int64_t)l * t.tchunks) * 32;
    tt = c0 + lane;
    nt = min(32, T - c0);
    valid = lane < nt;
  }
  const int4 d0 = __ldg(t.ldesc0 + l), d1 = __ldg(t.ldesc1 + l);
  const int32_t f = d0.x, to = d0.y, k = d0.z, fl = d0.w;
  const int32_t blo = min(f, to), bhi = max(f, to);
  const int32_t nl = d1.y - d1.x, nvt = __popc(fl & 15);
  const int32_t lenp = 1 + nl + (k >= 0 ? 1 : 0) + nvt, lenq = 1 + nl + nvt;
  const int32_t ccp = d1.z * T + tt, ccq = d1.w * T + tt;
  const int32_t off_v = 2 * t.G + 2 * t.L, off_th = off_v + t.N;
  if constexpr (STRUCT) {
    if (!valid) return;
    const int64_t posp = __ldg(t.colptr + ccp), posq = __ldg(t.colptr + ccq);
    int32_t jp = 0, jq = 0;
    rows[posp + jp++] = ccp;
    rows[posq + jq++] = ccq;
    for (int32_t a = d1.x; a < d1.y; ++a) {
      const int32_t l2 = __ldg(t.lnbx + a) >> 4;
      rows[posp + jp++] = __ldg(t.lent + 2 * t.G + l2) * T + tt;
      rows[posq + jq++] = __ldg(t.lent + 2 * t.G + t.L + l2) * T + tt;
    }
    if (k >= 0) rows[posp + jp++] = ccq;
    for (int i = 0; i < 4; ++i) {
      if (!(fl & (1 << i))) continue;
      const int32_t b = (i & 1) ? bhi : blo;
      const int32_t cr = __ldg(t.lent + ((i & 2) ? off_th : off_v) + b) * T + tt;
      rows[posp + jp++] = cr;
      rows[posq + jq++] = cr;
    }
    if (jp != lenp || jq != lenq || posp + jp != __ldg(t.colptr + ccp + 1) ||
        posq + jq != __ldg(t.colptr + ccq + 1))
      atomicOr(bad, 1);
    return;
  }
  double* stg = stg_all + warp * (kFLCap * 33);
  // ---- loads (every lane; invalid lanes clamp to the chunk's first period / the last item)
  const int32_t ts = (flat || valid) ? tt : c0, r = l * T + ts;
  const double G = __ldg(t.lg + l), B = __ldg(t.lb + l);
  const double vf = x[t.v0 + f * T + ts], vt = x[t.v0 + to * T + ts];
  const double thf = x[t.th0 + f * T + ts], tht = x[t.th0 + to * T + ts];
  const double xp = x[t.p0 + r], xq = x[t.q0 + r];
  const double dfp = dval(t, dv, t.flow_p0 + r), dfq = dval(t, dv, t.flow_q0 + r);
  const double dbp_lo = dval(t, dv, t.bal_p0 + blo * T + ts),
               dbp_hi = dval(t, dv, t.bal_p0 + bhi * T + ts);
  const double dbq_lo = dval(t, dv, t.bal_q0 + blo * T + ts),
               dbq_hi = dval(t, dv, t.bal_q0 + bhi * T + ts);
  const int32_t cps = d1.z * T + ts, cqs = d1.w * T + ts;
  const double sxp = sx[cps], sxq = sx[cqs];
  double wth = 0.0, dth = 0.0;
  if (k >= 0) {
    wth = w[t.therm0 + k * T + ts];
    dth = dval(t, dv, t.therm0 + k * T + ts);
  }
  const int2 cb = __ldg(t.lcb + l);
  int64_t basep = cb.x + (int64_t)c0 * lenp, baseq = cb.y + (int64_t)c0 * lenq;
  // flat lanes: the warp's p (q) columns are still one contiguous span of M (the columns of
  // consecutive (line, period) items are consecutive), with per-lane lengths -- staged in
  // output order at an exclusive prefix sum of the lengths, flushed as one stream
  int32_t offp = 0, offq = 0, totp = 0, totq = 0;
  bool staged = lenp <= kFLCap && lenq <= kFLCap;
  if constexpr (flat) {
    constexpr unsigned kAll = 0xffffffffu;
    const int32_t lp = valid ? lenp : 0, lq = valid ? lenq : 0;
    int32_t sp = lp, sq = lq;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const int32_t a = __shfl_up_sync(kAll, sp, dd), b = __shfl_up_sync(kAll, sq, dd);
      if (lane >= dd) {
        sp += a;
        sq += b;
      }
    }
    offp = sp - lp;
    offq = sq - lq;
    totp = __shfl_sync(kAll, sp, 31);
    totq = __shfl_sync(kAll, sq, 31);
    basep = __shfl_sync(kAll, cb.x + (int64_t)tt * lenp, 0);
    baseq = __shfl_sync(kAll, cb.y + (int64_t)tt * lenq, 0);
    staged = __all_sync(kAll, staged);
  }
  const LineState s = line_state(G, B, vf, vt, thf, tht);
  const double jtp = j_thermal(xp), jtq = j_thermal(xq);
  // ---- values, slot by slot; column p, then column q.  Staged (the common case:
  // both columns <= kFLCap slots) or written in place, a warp-uniform choice.
  auto columns = [&](auto staged) {
    constexpr bool ST = decltype(staged)::value;
    for (int Q = 0; Q < 2; ++Q) {
      const int64_t pos = ST ? 0 : (valid ? (int64_t)__ldg(t.colptr + (Q ? cqs : cps)) : 0);
      auto put = [&](int32_t j, double v) {
        if constexpr (ST && flat) {
          if (valid) stg[(Q ? offq : offp) + j] = v;
        } else if constexpr (ST) {
          stg[j * 33 + lane] = v;
        } else if (valid) {
          M[pos + j] = v;
        }
      };
      const double dlo = Q ? dbq_lo : dbp_lo, dhi = Q ? dbq_hi : dbp_hi, dfl = Q ? dfq : dfp;
      const double jt = Q ? jtq : jtp;
      const double sgn_lo = (fl & 16) ? 1.0 : -1.0, sgn_hi = (fl & 32) ? 1.0 : -1.0;
      {  // diagonal: thermal H (2w) then pairs bal(lo), bal(hi), flow, thermal, dw + Sx
        double acc = 0.0;
        if (k >= 0) acc += h_thermal_diag(wth);
        acc += pair_term(dlo, sgn_lo, sgn_lo);
        acc += pair_term(dhi, sgn_hi, sgn_hi);
        acc += pair_term(dfl, 1.0, 1.0);
        if (k >= 0) acc += pair_term(dth, jt, jt);
        acc += dw + (Q ? sxq : sxp);
        put(0, acc);
      }
      for (int32_t a = 0; a < nl; ++a) {  // flows l' > l sharing a bus: balance-row pairs
        const int32_t code = __ldg(t.lnbx + d1.x + a);
        double acc = 0.0;
        if (code & 1) acc += pair_term(dlo, (code & 4) ? 1.0 : -1.0, sgn_lo);
        if (code & 2) acc += pair_term(dhi, (code & 8) ? 1.0 : -1.0, sgn_hi);
        put(1 + a, acc);
      }
      int32_t j = 1 + nl;
      if (!Q && k >= 0) {  // (q(l), p(l)): thermal pair (2q)(2p)
        double acc = 0.0;
        acc += pair_term(dth, jtq, jtp);
        put(j++, acc);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // v(lo) v(hi) th(lo) th(hi): flow-row pairs
        if (!(fl & (1 << i))) continue;
        const int32_t b = (i & 1) ? bhi : blo;
        const int field = (i & 2) ? (b == f ? 3 : 4) : (b == f ? 1 : 2);
        double acc = 0.0;
        acc += pair_term(dfl, Q ? j_flow_q(s, G, B, field) : j_flow_p(s, G, B, field), 1.0);
        put(j++, acc);
      }
      if constexpr (ST && flat) {
        __syncwarp();
        const int32_t tot = Q ? totq : totp;
        double* o = M + (Q ? baseq : basep);
        for (int32_t e = lane; e < tot; e += 32) o[e] = stg[e];
        __syncwarp();
      } else if constexpr (ST) {
        warp_span_flush(M, Q ? baseq : basep, stg, Q ? lenq : lenp, nt, lane);
      }
    }
  };
  if (staged) columns(std::true_type{});
  else columns(std::false_type{});
}

// Grid-stride wrapper: `nvb` virtual CTAs on at most gridDim.x resident CTAs (the grid can be
// capped so that the latency-bound KKT kernels leave SM room for the callback stream).
template <bool STRUCT, bool FLAT>
__global__ void __launch_bounds__(kFLW * 32) k_fz_line(OpfKktTab t, int64_t nvb,
                                                      const double* __restrict__ x,
                                                      const double* __restrict__ w,
                                                      const double* __restrict__ sx, double dw,
                                                      const double* __restrict__ dv,
                                                      double* __restrict__ M,
                                                      int32_t* __restrict__ rows,
                                                      int32_t* __restrict__ bad) {
  fz_line_body<STRUCT, FLAT>(blockIdx.x, t, x, w, sx, dw, dv, M, rows, bad);
}
template <bool STRUCT, bool FLAT>
__global__ void __launch_bounds__(kFLW * 32, GN_FL_GS_MINB) k_fz_line_gs(OpfKktTab t, int64_t nvb,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ w,
                                                         const double* __restrict__ sx, double dw,
                                                         const double* __restrict__ dv,
                                                         double* __restrict__ M,
                                                         int32_t* __restrict__ rows,
                                                         int32_t* __restrict__ bad) {
  for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x)
    fz_line_body<STRUCT, FLAT>(vb, t, x, w, sx, dw, dv, M, rows, bad);
}

template <bool STRUCT>
__global__ void __launch_bounds__(256) k_fz_gen(OpfKktTab t, FIn in, const double* __restrict__ dv,
                                                double* __restrict__ M, int32_t* __restrict__ rows,
                                                int32_t* __restrict__ bad) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (int64_t)t.G * t.T) return;
  const int32_t g = (int32_t)(r / t.T), tt = (int32_t)(r - (int64_t)g * t.T);
  Ctx c{t, in, 0, tt, t.T, 0, 0, nullptr, 0, dv,
        0, t.G, 2 * t.G, 2 * t.G + t.L, 2 * t.G + 2 * t.L, 2 * t.G + 2 * t.L + t.N};
  fz_gen_cols<STRUCT>(c, g, M, rows, bad);
}

// ------------------------------------------------------ A straight from x
__device__ __forceinline__ void sj_row(const OpfKktTab& t, int32_t r, const double* __restrict__ x,
                                       double* __restrict__ dst) {
  const int32_t T = t.T;
  if (r < t.flow_p0) {  // balance rows: free generators (J = 1) then flows (J = +-1)
    const bool Q = r >= t.bal_q0;
    const int32_t rr = r - (Q ? t.bal_q0 : t.bal_p0);
    const int32_t b = rr / T;
    const int32_t nf = __ldg((Q ? t.ngq : t.ngp) + b);
    for (int32_t i = 0; i < nf; ++i) dst[i] = 0.0 + 1.0;
    const int32_t b0 = __ldg(t.bl_ptr + b), b1 = __ldg(t.bl_ptr + b + 1);
    for (int32_t i = b0; i < b1; ++i) dst[nf + (i - b0)] = 0.0 + ((__ldg(t.bl + i) & 1) ? -1.0 : 1.0);
  } else if (r < t.therm0) {  // flow definitions: J from the line state
    const bool Q = r >= t.flow_q0;
    const int32_t rr = r - (Q ? t.flow_q0 : t.flow_p0);
    const int32_t l = rr / T, tt = rr - l * T;
    const int32_t f = __ldg(t.lf + l), to = __ldg(t.lt + l);
    const double G = __ldg(t.lg + l), B = __ldg(t.lb + l);
    const LineState s = line_state(G, B, x[t.v0 + (int64_t)f * T + tt], x[t.v0 + (int64_t)to * T + tt],
                                   x[t.th0 + (int64_t)f * T + tt], x[t.th0 + (int64_t)to * T + tt]);
#pragma unroll
    for (int fl = 0; fl < 5; ++fl) {
      const int p = __ldg(t.fpos + 5 * l + fl);
      if (p >= 0) dst[p] = 0.0 + (Q ? j_flow_q(s, G, B, fl) : j_flow_p(s, G, B, fl));
    }
  } else if (r < t.ang0) {  // thermal [p, q]: (2p, 2q)
    const int32_t rr = r - t.therm0, k = rr / T, tt = rr - k * T;
    const int32_t l = __ldg(t.th_line + k);
    dst[0] = 0.0 + j_thermal(x[t.p0 + (int64_t)l * T + tt]);
    dst[1] = 0.0 + j_thermal(x[t.q0 + (int64_t)l * T + tt]);
  } else if (r < t.ramp0) {  // angle [th_f, th_t]: (1, -1)
    const int32_t l = (r - t.ang0) / T;
    const int pf = __ldg(t.apos + 2 * l), pt = __ldg(t.apos + 2 * l + 1);
    if (pf >= 0) dst[pf] = 0.0 + 1.0;
    if (pt >= 0) dst[pt] = 0.0 + (-1.0);
  } else {  // ramp [pg_{s-1}, pg_s]: (-1, 1); a shard's first row keeps pg_s only
    const int32_t len = __ldg(t.rowptr + r + 1) - __ldg(t.rowptr + r);
    if (len == 2) {
      dst[0] = 0.0 + (-1.0);
      dst[1] = 0.0 + 1.0;
    } else if (len == 1) {
      dst[0] = 0.0 + 1.0;
    }
  }
}

// A = set_jacobian(eval_jac(x)) straight from x, one warp per task.  The rows of
// one entity over consecutive periods are consecutive CSR rows, i.e. one
// contiguous span of A, and every span is written coalesced:
//   * balance rows of a bus (all periods): constants (+1 per free generator,
//     +-1 per incident line, held by lane j = slot j and broadcast by shuffle);
//   * flow_p and flow_q rows of (line, 32 periods): the line state is computed
//     once for both rows, staged ([slot][lane]) and written back;
//   * thermal rows of (thermal line, 32 periods): (2p, 2q), lane = period;
//   * angle rows of a line (all periods): (+1, -1) at the free angle slots;
//   * ramp rows: one thread per row.
// the A kernel's own grid cap under a capped KKT (tuning builds; 0 = the KKT's cap)
#ifndef GN_SJ_CAP
#define GN_SJ_CAP 0
#endif
#ifndef GN_SJW
#define GN_SJW 8
#endif
constexpr int kSJW = GN_SJW;  // warps per CTA
template <bool FLAT>
__device__ __forceinline__ void set_jac_body(int64_t vblock, const OpfKktTab& t, int32_t m,
                                             const double* __restrict__ x,
                                             double* __restrict__ A, int skip_flow) {
  __shared__ double stg_all[kSJW * 5 * 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t T = t.T, tch = t.tchunks;
  const int32_t LT = (t.ang0 - t.therm0) / (T > 0 ? T : 1);
  int64_t wg = vblock * kSJW + warp;
  if (wg < 2ll * t.N) {  // balance rows of bus b, all periods
    const bool Q = wg >= t.N;
    const int32_t b = (int32_t)(wg - (Q ? t.N : 0));
    const int32_t nf = __ldg((Q ? t.ngq : t.ngp) + b);
    const int32_t b0 = __ldg(t.bl_ptr + b), len = nf + __ldg(t.bl_ptr + b + 1) - b0;
    if (len == 0) return;
    const int64_t base = __ldg(t.rbase + (Q ? t.N : 0) + b);
    if (len > 32) {  // (very high degree: slot by slot)
      for (int32_t e = lane; e < T * len; e += 32) {
        const int32_t j = e % len;
        A[base + e] = j < nf ? 0.0 + 1.0 : 0.0 + ((__ldg(t.bl + b0 + j - nf) & 1) ? -1.0 : 1.0);
      }
      return;
    }
    double v = 0.0 + 1.0;
    if (lane >= nf && lane < len) v = 0.0 + ((__ldg(t.bl + b0 + lane - nf) & 1) ? -1.0 : 1.0);
    warp_const_rows(A, base, v, len, T, lane);
    return;
  }
  wg -= 2ll * t.N;
  const int64_t nflow = skip_flow ? 0 : (FLAT ? ((int64_t)t.L * T + 31) / 32 : (int64_t)t.L * tch);
  if (FLAT && wg < nflow) {  // flow_p / flow_q rows of 32 flat (line, period) items
    constexpr unsigned kAll = 0xffffffffu;
    double* stg = stg_all + warp * (5 * 33);
    const int64_t nitems = (int64_t)t.L * T, item = wg * 32 + lane;
    const bool valid = item < nitems;
    const int64_t it = valid ? item : nitems - 1;
    const int32_t l = (int32_t)(it / T), ts = (int32_t)(it - (int64_t)l * T);
    const int4 d0 = __ldg(t.ldesc0 + l);
    const int32_t f = d0.x, to = d0.y, len = 1 + __popc(d0.w & 15);
    const double G = __ldg(t.lg + l), B = __ldg(t.lb + l);
    const LineState s = line_state(G, B, x[t.v0 + f * T + ts], x[t.v0 + to * T + ts],
                                   x[t.th0 + f * T + ts], x[t.th0 + to * T + ts]);
    // consecutive items are consecutive CSR rows: one span per row type, per-lane lengths
    const int32_t lv = valid ? len : 0;
    int32_t sc = lv;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const int32_t a = __shfl_up_sync(kAll, sc, dd);
      if (lane >= dd) sc += a;
    }
    const int32_t off = sc - lv, tot = __shfl_sync(kAll, sc, 31);
    const int64_t bp = __shfl_sync(kAll, __ldg(t.rbase + 2 * t.N + l) + (int64_t)ts * len, 0);
    const int64_t bq = __shfl_sync(kAll, __ldg(t.rbase + 2 * t.N + t.L + l) + (int64_t)ts * len, 0);
    int pos[5];
#pragma unroll
    for (int fl = 0; fl < 5; ++fl) pos[fl] = __ldg(t.fpos + 5 * l + fl);
#pragma unroll
    for (int Q = 0; Q < 2; ++Q) {
      if (valid) {
#pragma unroll
        for (int fl = 0; fl < 5; ++fl)
          if (pos[fl] >= 0) stg[off + pos[fl]] = 0.0 + (Q ? j_flow_q(s, G, B, fl) : j_flow_p(s, G, B, fl));
      }
      __syncwarp();
      double* o = A + (Q ? bq : bp);
      for (int32_t e = lane; e < tot; e += 32) o[e] = stg[e];
      __syncwarp();
    }
    return;
  }
  if (!FLAT && wg < nflow) {  // flow_p / flow_q rows of (line, 32 periods)
    double* stg = stg_all + warp * (5 * 33);
    const int32_t l = (int32_t)(wg / tch), c0 = (int32_t)(wg - (int64_t)l * tch) * 32;
    const int32_t nt = min(32, T - c0), ts = lane < nt ? c0 + lane : c0;
    const int4 d0 = __ldg(t.ldesc0 + l);
    const int32_t f = d0.x, to = d0.y, len = 1 + __popc(d0.w & 15);
    const double G = __ldg(t.lg + l), B = __ldg(t.lb + l);
    const LineState s = line_state(G, B, x[t.v0 + f * T + ts], x[t.v0 + to * T + ts],
                                   x[t.th0 + f * T + ts], x[t.th0 + to * T + ts]);
    const int64_t bp = __ldg(t.rbase + 2 * t.N + l) + (int64_t)c0 * len;
    const int64_t bq = __ldg(t.rbase + 2 * t.N + t.L + l) + (int64_t)c0 * len;
    int pos[5];
#pragma unroll
    for (int fl = 0; fl < 5; ++fl) pos[fl] = __ldg(t.fpos + 5 * l + fl);
#pragma unroll
    for (int fl = 0; fl < 5; ++fl)
      if (pos[fl] >= 0) stg[pos[fl] * 33 + lane] = 0.0 + j_flow_p(s, G, B, fl);
    warp_span_flush(A, bp, stg, len, nt, lane);
#pragma unroll
    for (int fl = 0; fl < 5; ++fl)
      if (pos[fl] >= 0) stg[pos[fl] * 33 + lane] = 0.0 + j_flow_q(s, G, B, fl);
    warp_span_flush(A, bq, stg, len, nt, lane);
    return;
  }
  wg -= nflow;
  const int64_t nth = FLAT ? ((int64_t)LT * T + 31) / 32 : LT;
  if (FLAT && wg < nth) {  // thermal rows of 32 flat (slot, period) items: (2p, 2q) each
    const int64_t item = wg * 32 + lane;
    if (item >= (int64_t)LT * T) return;
    const int32_t k = (int32_t)(item / T), tt = (int32_t)(item - (int64_t)k * T);
    const int32_t l = __ldg(t.th_line + k);
    const double pv = x[t.p0 + (int64_t)l * T + tt], qv = x[t.q0 + (int64_t)l * T + tt];
    double* dst = A + __ldg(t.rbase + 2 * t.N + 2 * t.L + k) + 2LL * tt;
    dst[0] = 0.0 + j_thermal(pv);
    dst[1] = 0.0 + j_thermal(qv);
    return;
  }
  if (!FLAT && wg < LT) {  // thermal rows of thermal slot k, all periods: [p, q] -> (2p, 2q)
    const int32_t k = (int32_t)wg, l = __ldg(t.th_line + k);
    const int64_t base = __ldg(t.rbase + 2 * t.N + 2 * t.L + k);
    const double* xp = x + t.p0 + l * T;
    const double* xq = x + t.q0 + l * T;
    constexpr int kU = 4;  // periods per lane per round: all loads of a round, then its stores
    for (int32_t c0 = 0; c0 < T; c0 += 32 * kU) {
      double pv[kU], qv[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const int32_t tt = c0 + 32 * j + lane;
        pv[j] = tt < T ? xp[tt] : 0.0;
        qv[j] = tt < T ? xq[tt] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const int32_t tt = c0 + 32 * j + lane;
        if (tt < T) {
          A[base + 2 * tt] = 0.0 + j_thermal(pv[j]);
          A[base + 2 * tt + 1] = 0.0 + j_thermal(qv[j]);
        }
      }
    }
    return;
  }
  wg -= nth;
  if (wg < t.L) {  // angle rows of line l, all periods: [th_f, th_t] -> (1, -1)
    const int32_t l = (int32_t)wg;
    const int pf = __ldg(t.apos + 2 * l), pt = __ldg(t.apos + 2 * l + 1);
    const int32_t len = (pf >= 0) + (pt >= 0);
    if (len == 0) return;
    const int64_t base = __ldg(t.rbase + 2 * t.N + 2 * t.L + LT + l);
    const double v = lane == pf ? 0.0 + 1.0 : 0.0 + (-1.0);
    warp_const_rows(A, base, v, len, T, lane);
    return;
  }
  wg -= t.L;
  const int64_t r = (int64_t)t.ramp0 + wg * 32 + lane;  // ramp rows, one thread each
  if (r >= m) return;
  const int32_t ri = (int32_t)r;
  double* dst = A + __ldg(t.rowptr + ri);
  // [pg_{s-1}, pg_s]: (-1, 1); a shard's first row keeps pg_s only
  const int32_t len = __ldg(t.rowptr + ri + 1) - __ldg(t.rowptr + ri);
  if (len == 2) {
    dst[0] = 0.0 + (-1.0);
    dst[1] = 0.0 + 1.0;
  } else if (len == 1) {
    dst[0] = 0.0 + 1.0;
  }
}

template <bool FLAT>
__global__ void __launch_bounds__(kSJW * 32, GN_SJ_MINB) k_opf_set_jac_fused(OpfKktTab t, int64_t nvb,
                                                                int32_t m,
                                                                const double* __restrict__ x,
                                                                double* __restrict__ A,
                                                                int skip_flow) {
  set_jac_body<FLAT>(blockIdx.x, t, m, x, A, skip_flow);
}
template <bool FLAT>
__global__ void __launch_bounds__(kSJW * 32, GN_SJ_GS_MINB) k_opf_set_jac_fused_gs(OpfKktTab t, int64_t nvb,
                                                                   int32_t m,
                                                                   const double* __restrict__ x,
                                                                   double* __restrict__ A,
                                                                   int skip_flow) {
  for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) set_jac_body<FLAT>(vb, t, m, x, A, skip_flow);
}

// ------------------------------------------------------------------ host
// Auxiliary streams of the fork/join below (created on first use, same priority as the
// KKT stream); false when kernels must run serially (per-kernel profiling).
static bool ensure_aux(gn_kkt* K) {
  if (profiling()) return false;
  OpfKkt* X = K->opf;
  int prio = 0;
  GN_CK(cudaStreamGetPriority(K->stream, &prio));
  if (!X->aux[0] || prio != X->aux_prio) {
    for (auto& a : X->aux) {
      if (a) GN_CK(cudaStreamDestroy(a));
      GN_CK(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, prio));
    }
    if (!X->ev_fork) {
      GN_CK(cudaEventCreateWithFlags(&X->ev_fork, cudaEventDisableTiming));
      GN_CK(cudaEventCreateWithFlags(&X->ev_fork2, cudaEventDisableTiming));
      for (auto& e : X->ev_join) GN_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    X->aux_prio = prio;
  }
  return true;
}

// The column kernels write disjoint parts of M.  In value mode the bus classes are forked
// over auxiliary streams (fork/join by events: capturable in a CUDA graph) beside the
// flow-column kernel on the KKT stream, so the short, low-occupancy degree-class launches
// overlap it instead of each paying its own tail.  Per-kernel profiling runs them serially.
// Bus-class lanes: one for large problems (the classes are long and fill the SMs; more
// concurrent KKT kernels only crowd out the flow-column kernel and the callback stream),
// four when the whole bus sweep is a few thousand warps (the step is then the chain of
// short latency-bound launches, which parallel lanes shorten).  Measured, step ms for
// 1 / 2 / 4 / 8 lanes: 1354 x 24: 0.059 / 0.058 / 0.044 / 0.050; 9241 x 48: 0.255 /
// 0.270 / 0.274 / 0.274; 30k x 96: 1.179 / 1.190 / 1.217 / 1.246.  Re-measured on the final
// kernels: 9241 x 48 1 / 2 / 3 lanes 0.2335 / 0.238 / 0.248; 30k x 96 1 / 2: 1.111 / 1.140.
// GRIDNLP_B200_BUS_LANES overrides (1 .. kBusClasses).
static int bus_lanes(const OpfKkt* X) {
  static const int env = [] {
    const char* e = std::getenv("GRIDNLP_B200_BUS_LANES");
    return e ? std::atoi(e) : 0;
  }();
  if (env > 0) return env < kBusClasses ? env : kBusClasses;
  int64_t warps = 0;
  for (int k = 0; k < kBusClasses; ++k) warps += (int64_t)X->n_bus_cls[k] * X->t.tchunks;
  return warps <= 4096 ? 4 : 1;
}

#ifndef GN_GEN_LANE
#define GN_GEN_LANE 1
#endif
template <bool STRUCT>
static void launch_fused(gn_kkt* K, const FIn& in, const double* dv, double* M, int32_t* rows,
                         int32_t* bad) {
  OpfKkt* X = K->opf;
  const OpfKktTab& t = X->t;
  cudaStream_t s = K->stream;
  const bool fork = !STRUCT && ensure_aux(K);
  const int nlanes = fork ? bus_lanes(X) : 1;
  if (fork) {
    GN_CK(cudaEventRecord(X->ev_fork, s));
    for (int a = 0; a < nlanes; ++a) GN_CK(cudaStreamWaitEvent(X->aux[a], X->ev_fork, 0));
  }
  // degree classes 1..kBusRegMax, le8, rest: round-robin over the lanes, largest first
  // (d3, d4, d2, d5 .. rest, then d1)
  for (int i = 0; i < kBusClasses; ++i) {
    const int k = i < 3 ? (i == 0 ? 2 : i == 1 ? 3 : 1) : (i == kBusClasses - 1 ? 0 : i + 1);
    launch_fz_bus(t, X->bus_cls[k].p, X->n_bus_cls[k],
                  k < kBusRegMax ? k + 1 : (k == kBusRegMax ? 8 : X->maxdeg_rest), k, in, dv, M,
                  rows, bad, fork ? X->aux[i % nlanes] : s);
  }
  const int64_t nl = (int64_t)t.L * t.T, ng = (int64_t)t.G * t.T;
  if (nl > 0) {
    KTimer kt("k_fz_line", s);
    const bool flat = !STRUCT && GN_FL_FLAT && (t.T % 32) != 0;
    const int64_t warps = flat ? (nl + 31) / 32 : (int64_t)t.L * t.tchunks;
    const int64_t nvb = (warps + kFLW - 1) / kFLW;
    const unsigned g = grid_cap(nvb, t.grid_cap);
    if (flat) {
      if (g < nvb)  // capped grid: the grid-stride variant
        k_fz_line_gs<STRUCT, true><<<g, kFLW * 32, 0, s>>>(t, nvb, in.x, in.w, in.sx, in.dw, dv, M, rows, bad);
      else
        k_fz_line<STRUCT, true><<<g, kFLW * 32, 0, s>>>(t, nvb, in.x, in.w, in.sx, in.dw, dv, M, rows, bad);
    } else {
      if (g < nvb)
        k_fz_line_gs<STRUCT, false><<<g, kFLW * 32, 0, s>>>(t, nvb, in.x, in.w, in.sx, in.dw, dv, M, rows, bad);
      else
        k_fz_line<STRUCT, false><<<g, kFLW * 32, 0, s>>>(t, nvb, in.x, in.w, in.sx, in.dw, dv, M, rows, bad);
    }
    count_launch();
  }
  // the generator columns: on their own auxiliary lane beside the flow-column kernel for
  // large sweeps (one bus lane; 30k x 96 -0.2%), else after it on the KKT stream (on the
  // small, four-lane sweeps a fifth stream costs 2%)
  const bool gen_lane = fork && GN_GEN_LANE && nlanes == 1;
  cudaStream_t sg = gen_lane ? X->aux[kBusClasses - 1] : s;
  if (gen_lane) GN_CK(cudaStreamWaitEvent(sg, X->ev_fork, 0));
  if (ng > 0) {
    KTimer kt("k_fz_gen", sg);
    k_fz_gen<STRUCT><<<(unsigned)((ng + 255) / 256), 256, 0, sg>>>(t, in, dv, M, rows, bad);
    count_launch();
  }
  if (fork) {
    for (int a = 0; a < nlanes; ++a) {
      GN_CK(cudaEventRecord(X->ev_join[a], X->aux[a]));
      GN_CK(cudaStreamWaitEvent(s, X->ev_join[a], 0));
    }
    if (gen_lane) {
      GN_CK(cudaEventRecord(X->ev_join[kBusClasses - 1], sg));
      GN_CK(cudaStreamWaitEvent(s, X->ev_join[kBusClasses - 1], 0));
    }
  }
  GN_CK(cudaGetLastError());
}

bool opf_fused_ready(const gn_kkt* K) { return K->opf && K->opf->fused_ready; }

void launch_dvec(gn_kkt* K, const double* ss, double dw, double dc) {
  if (K->m <= 0) return;
  KTimer kt("k_fz_dvec", K->stream);
  k_fz_dvec<<<(unsigned)((K->m + 1023) / 1024), 256, 0, K->stream>>>(K->m, ss, dw, dc, K->dvals.p);
  count_launch();
}

void opf_assemble_fused(gn_kkt* K, const double* x, const double* w, double ow, const double* sx,
                        const double* ss, double dw, double dc) {
  FIn in{x, w, ow, sx, ss, dw, dc};
  K->opf->t.kdw = dw;
  K->opf->t.kdc = dc;
#if GN_DV_INLINE
  launch_fused<false>(K, in, ss, K->mvals.p, nullptr, nullptr);
#else
  launch_dvec(K, ss, dw, dc);
  launch_fused<false>(K, in, K->dvals.p, K->mvals.p, nullptr, nullptr);
#endif
}

static void set_jac_launch(gn_kkt* K, const double* x, int skip_flow, cudaStream_t st) {
  const OpfKktTab& t = K->opf->t;
  if (K->m <= 0) return;
  {
    KTimer kt(skip_flow ? "k_opf_set_jac_fused<noflow>" : "k_opf_set_jac_fused", st);
    const int64_t LT = t.T > 0 ? (t.ang0 - t.therm0) / t.T : 0;
    // flat (entity, period) lanes for the flow and thermal rows when T leaves lanes idle
    const bool flat = GN_FL_FLAT && (t.T % 32) != 0;
    const int64_t nflow = skip_flow ? 0 : (flat ? ((int64_t)t.L * t.T + 31) / 32
                                                : (int64_t)t.L * t.tchunks);
    const int64_t nth = flat ? (LT * t.T + 31) / 32 : LT;
    const int64_t warps = 2ll * t.N + nflow + nth + t.L + (K->m - t.ramp0 + 31) / 32;
    const int64_t nvb = (warps + kSJW - 1) / kSJW;
    const unsigned g = grid_cap(nvb, (GN_SJ_CAP > 0 && t.grid_cap > 0) ? GN_SJ_CAP : t.grid_cap);
    if (flat) {
      if (g < nvb)
        k_opf_set_jac_fused_gs<true><<<g, kSJW * 32, 0, st>>>(t, nvb, K->m, x, K->avals.p, skip_flow);
      else
        k_opf_set_jac_fused<true><<<g, kSJW * 32, 0, st>>>(t, nvb, K->m, x, K->avals.p, skip_flow);
    } else {
      if (g < nvb)
        k_opf_set_jac_fused_gs<false><<<g, kSJW * 32, 0, st>>>(t, nvb, K->m, x, K->avals.p, skip_flow);
      else
        k_opf_set_jac_fused<false><<<g, kSJW * 32, 0, st>>>(t, nvb, K->m, x, K->avals.p, skip_flow);
    }
  }
  count_launch();
  GN_CK(cudaGetLastError());
}

void opf_set_jacobian_fused(gn_kkt* K, const double* x) { set_jac_launch(K, x, 0, K->stream); }

// set_jacobian_x + assemble_x at the same x (gn_kkt_update_x).  (Writing A's flow rows
// from the flow-column kernel's line state was measured slower than the separate
// set_jacobian pass: it costs that latency-bound kernel a third of its occupancy.)
void opf_update_fused(gn_kkt* K, const double* x, const double* w, double ow, const double* sx,
                      const double* ss, double dw, double dc) {
  // A (set_jacobian) and M (assemble) are independent given x: A is built on a third
  // auxiliary stream beside the M kernels, so the two latency-bound phases overlap
  OpfKkt* X = K->opf;
  static const bool fork_sj = [] {
    const char* e = std::getenv("GRIDNLP_B200_SETJAC_FORK");
    return !e || std::atoi(e) != 0;
  }();
  if (fork_sj && ensure_aux(K)) {
    GN_CK(cudaEventRecord(X->ev_fork2, K->stream));
    cudaStream_t sj = X->aux[OpfKkt::kAuxSetJac];
    GN_CK(cudaStreamWaitEvent(sj, X->ev_fork2, 0));
    set_jac_launch(K, x, 0, sj);
    GN_CK(cudaEventRecord(X->ev_join[OpfKkt::kAuxSetJac], sj));
    opf_assemble_fused(K, x, w, ow, sx, ss, dw, dc);
    GN_CK(cudaStreamWaitEvent(K->stream, X->ev_join[OpfKkt::kAuxSetJac], 0));
  } else {
    set_jac_launch(K, x, 0, K->stream);
    opf_assemble_fused(K, x, w, ow, sx, ss, dw, dc);
  }
}

// Structure check of the fused enumeration (row index of every slot, column lengths).
bool opf_fused_verify(gn_kkt* K) {
  const OpfKktTab& t = K->opf->t;
  if (!fz_bus_fits(t.maxdeg)) return false;  // one line per lane, one warp's shared memory
  cudaStream_t s = K->stream;
  DBuf<int32_t> rows, bad, diff;
  rows.alloc(static_cast<size_t>(K->mnnz) + 1);
  bad.alloc(1);
  diff.alloc(1);
  GN_CK(cudaMemsetAsync(bad.p, 0, 4, s));
  GN_CK(cudaMemsetAsync(diff.p, 0, 4, s));
  GN_CK(cudaMemsetAsync(rows.p, 0xff, sizeof(int32_t) * K->mnnz, s));
  FIn in{};
  launch_fused<true>(K, in, nullptr, nullptr, rows.p, bad.p);
  int32_t owned_nnz = 0;  // slots of the owned columns (next-ghost columns are not assembled)
  GN_CK(cudaMemcpyAsync(&owned_nnz, K->M.ptr.p + t.n_owned, 4, cudaMemcpyDeviceToHost, s));
  GN_CK(cudaStreamSynchronize(s));
  count_diff(rows.p, K->M.idx.p, owned_nnz, diff.p, s);
  int32_t hb[2] = {0, 0};
  GN_CK(cudaMemcpyAsync(&hb[0], bad.p, 4, cudaMemcpyDeviceToHost, s));
  GN_CK(cudaMemcpyAsync(&hb[1], diff.p, 4, cudaMemcpyDeviceToHost, s));
  GN_CK(cudaStreamSynchronize(s));
  return hb[0] == 0 && hb[1] == 0;
}

}  // namespace gnb
