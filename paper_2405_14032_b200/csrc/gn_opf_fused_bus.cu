// Fused bus-column kernel: the v(n) and th(n) columns of M from x.
//
// A warp owns one bus n and 32/P consecutive periods; lane = (period group g,
// line slot i), P = next power of two >= deg(n).  Lane (g, i) evaluates the
// trigonometric state of the bus's i-th incident line (ascending l) at period
// t0 + g once, and from it the 26 contributor terms that line adds to the slots
// of v(n) and th(n).  Every slot is then one ordered reduction over the line
// lanes of its group (warp shuffles), reproducing CondensedKkt::assemble's
// summation order exactly (condensed.hpp:118-134):
//
//   v(n) column, rows ascending
//     (v_n, v_n)     Hp(1,1|2,2)... Hq ...  pairs flow_p ... flow_q ...  + dw + Sx
//     (v_n', v_n)    per neighbour n' > n: Hp(2,1), Hq(2,1), pair_p, pair_q over its lines
//     (th_x, v_n)    x in {n} U neighbours ascending (slots (3,1)/(4,2) and (4,1)/(3,2))
//   th(n) column
//     (th_n, th_n)   Hp(3,3|4,4), Hq, pairs flow_p, flow_q, angle  + dw + Sx
//     (th_n', th_n)  per neighbour n' > n: Hp(4,3), Hq(4,3), pair_p, pair_q, pair_angle
//
// Hessian slots that are structurally zero are added as +0.0, a no-op on an
// accumulator that starts at +0.0 (it never becomes -0.0).
#include <cstdlib>
#include <mutex>
#include <vector>

#include "gn_opf_kkt.cuh"

// (the STRUCT instantiations return before the value code: "loop is not reachable")
#pragma nv_diag_suppress 128
#include "gn_opf_math.cuh"

namespace gnb {

// multiplier of the KKT grid cap for the register-resident bus classes (tuning builds)
#ifndef GN_BUSR_CAP_MUL
#define GN_BUSR_CAP_MUL 1
#endif
#ifndef GN_BW3
#define GN_BW3 4
#endif
#ifndef GN_BUSR_FLAT
#define GN_BUSR_FLAT 1  // register classes: flat (bus, period) lanes; 0: a warp per (bus, 32 t)
#endif
constexpr int kBW3 = GN_BW3;  // warps per CTA
// resident CTAs per SM the register allocation of k_fz_busr<DEG> must allow
// (per degree: overridable one by one in tuning builds, GN_BUSR_MINB_D<k>)
#ifndef GN_BUSR_MINB_D1
#define GN_BUSR_MINB_D1 8
#endif
#ifndef GN_BUSR_MINB_D2
#define GN_BUSR_MINB_D2 5
#endif
#ifndef GN_BUSR_MINB_D3
#define GN_BUSR_MINB_D3 3
#endif
#ifndef GN_BUSR_MINB_D4
#define GN_BUSR_MINB_D4 3
#endif
#ifndef GN_BUSR_MINB_D5
#define GN_BUSR_MINB_D5 2
#endif
#ifndef GN_BUSR_MINB_D6
#define GN_BUSR_MINB_D6 2
#endif
#ifndef GN_BUSR_MINB_D7
#define GN_BUSR_MINB_D7 1
#endif
constexpr int kBusrMinBlocks[10] = {1, GN_BUSR_MINB_D1, GN_BUSR_MINB_D2, GN_BUSR_MINB_D3,
                                    GN_BUSR_MINB_D4, GN_BUSR_MINB_D5, GN_BUSR_MINB_D6,
                                    GN_BUSR_MINB_D7, GN_BUSR_MINB_D7, GN_BUSR_MINB_D7};
constexpr int kSV = 11;
constexpr int kBusSmemMax = 200 * 1024;  // dynamic shared memory cap of the bus kernel  // shared doubles per (line, lane): Cs Sn cs sn vf vt w7 w8 d7 d8 d10

// One warp per (bus n, 32 consecutive periods), lane = period.  The
// trigonometric state (Cs, Sn, cs, sn) of each incident line is computed once
// per lane into shared memory; the bus's slot program (host-built: lane mask of
// the lines of each slot + slot type) then drives the ordered sums.
template <bool STRUCT>
__global__ void __launch_bounds__(kBW3 * 32, 3) k_fz_bus3(OpfKktTab t, const int4* __restrict__ buses,
                                                       int32_t n_buses, int32_t maxdeg, FIn in,
                                                       const double* __restrict__ dv,
                                                       double* __restrict__ M,
                                                       int32_t* __restrict__ rows,
                                                       int32_t* __restrict__ bad) {
  extern __shared__ double bsm[];
  const int nw = blockDim.x >> 5;  // warps per CTA (fewer for very-high-degree classes)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * nw + warp;
  const int64_t n64 = w / t.tchunks;
  if (n64 >= n_buses) return;  // warp-uniform
  const int4 bd0 = __ldg(buses + kBusDesc * n64), bd1 = __ldg(buses + kBusDesc * n64 + 1);
  const int4 bd2 = __ldg(buses + kBusDesc * n64 + 2);
  const int32_t n = bd0.x, b0 = bd0.y, deg = bd0.z & 255, T = t.T;
  const int32_t tt = (int32_t)(w - n64 * t.tchunks) * 32 + lane;
  // per (line, lane): 6 state values + the 5 row inputs it contributes with
  double* S = bsm + (size_t)warp * maxdeg * kSV * 32 + lane;
  // per-line warp-uniform data, filled by lanes 0..deg-1 in parallel
  struct LU {
    double G, B;
    int32_t l, fr;
  };
  LU* U = reinterpret_cast<LU*>(bsm + (size_t)nw * maxdeg * kSV * 32) + warp * maxdeg;
  if (lane < deg) {
    const int2 e = __ldg(t.blx + b0 + lane);
    const double2 gb = __ldg(t.blgb + b0 + lane);
    U[lane] = LU{gb.x, gb.y, e.x >> 1, e.x & 1};
  }
  __syncwarp();
  if (tt >= T) return;  // no warp collectives below
  const int32_t off_v = 2 * t.G + 2 * t.L, off_th = off_v + t.N;

  if constexpr (!STRUCT) {
    // every global input of the slot program is read exactly once, up front
    // (independent loads in flight together); the slot loop reads only smem
#pragma unroll 4
    for (int i = 0; i < deg; ++i) {
      const int2 e = __ldg(t.blx + b0 + i);
      const double2 gb = __ldg(t.blgb + b0 + i);
      const int32_t l = e.x >> 1, f = (e.x & 1) ? n : e.y, to = (e.x & 1) ? e.y : n;
      const int32_t rl = l * T + tt;
      const double w7 = in.w[t.flow_p0 + rl], w8 = in.w[t.flow_q0 + rl];
      const double d7 = dval(t, dv, t.flow_p0 + rl), d8 = dval(t, dv, t.flow_q0 + rl),
                   d10 = dval(t, dv, t.ang0 + rl);
      const LineState s = line_state(gb.x, gb.y, in.x[t.v0 + f * T + tt], in.x[t.v0 + to * T + tt],
                                     in.x[t.th0 + f * T + tt], in.x[t.th0 + to * T + tt]);
      double* q = S + (size_t)i * kSV * 32;
      q[0 * 32] = s.Cs;
      q[1 * 32] = s.Sn;
      q[2 * 32] = s.cs;
      q[3 * 32] = s.sn;
      q[4 * 32] = s.vf;
      q[5 * 32] = s.vt;
      q[6 * 32] = w7;
      q[7 * 32] = w8;
      q[8 * 32] = d7;
      q[9 * 32] = d8;
      q[10 * 32] = d10;
    }
  }
  // line k of the bus: state + the per-row inputs of this period
  struct LV {
    LineState s;
    double G, B;
    double w7, w8, d7, d8, d10;
    int32_t l, fr;
  };
  auto lv = [&](int k) {
    LV r;
    const LU u = U[k];
    r.l = u.l;
    r.fr = u.fr;
    r.G = u.G;
    r.B = u.B;
    const double* q = S + (size_t)k * kSV * 32;
    r.s.Cs = q[0 * 32];
    r.s.Sn = q[1 * 32];
    r.s.cs = q[2 * 32];
    r.s.sn = q[3 * 32];
    r.s.vf = q[4 * 32];
    r.s.vt = q[5 * 32];
    r.s.vfvt = r.s.vf * r.s.vt;
    r.w7 = q[6 * 32];
    r.w8 = q[7 * 32];
    r.d7 = q[8 * 32];
    r.d8 = q[9 * 32];
    r.d10 = q[10 * 32];
    return r;
  };
  auto w7 = [](const LV& r) { return r.w7; };
  auto w8 = [](const LV& r) { return r.w8; };
  auto d7 = [](const LV& r) { return r.d7; };
  auto d8 = [](const LV& r) { return r.d8; };
  auto d10 = [](const LV& r) { return r.d10; };
  // fields of this bus's side (n = from -> v_f / th_f)
  auto JP = [&](const LV& r, bool other, bool theta) {
    const int f = theta ? ((r.fr ^ other) ? 3 : 4) : ((r.fr ^ other) ? 1 : 2);
    return j_flow_p(r.s, r.G, r.B, f);
  };
  auto JQ = [&](const LV& r, bool other, bool theta) {
    const int f = theta ? ((r.fr ^ other) ? 3 : 4) : ((r.fr ^ other) ? 1 : 2);
    return j_flow_q(r.s, r.G, r.B, f);
  };

  auto col = [&](int32_t off, int32_t e) {
    const int32_t k = __ldg(t.lent + off + e);
    return k < 0 ? -1 : k * T + tt;
  };
  const int32_t cv = bd1.x < 0 ? -1 : bd1.x * T + tt, ct = bd1.y < 0 ? -1 : bd1.y * T + tt;
  const int64_t posv = cv >= 0 ? (int64_t)bd2.x + (int64_t)tt * bd2.y : 0;
  const int64_t post = ct >= 0 ? (int64_t)bd2.z + (int64_t)tt * bd2.w : 0;
  int jv = 0, jt = 0;
  const int32_t p0 = bd0.w, p1 = p0 + (bd0.z >> 8);
#define PASS(expr)                                 \
  for (uint32_t mm = mask; mm; mm &= mm - 1) {     \
    const LV r = lv(__ffs(mm) - 1);                \
    acc += (expr);                                 \
  }
  // loop-invariant / next-iteration global loads issued ahead of their use
  const double sxv = (!STRUCT && cv >= 0) ? in.sx[cv] : 0.0;
  const double sxt = (!STRUCT && ct >= 0) ? in.sx[ct] : 0.0;
  unsigned long long code_next = p0 < p1 ? __ldg(t.bprog + p0) : 0ull;
  // The three own slots (v,v) (th,v) (th,th) run over every incident line with
  // the same pass structure: one fused sweep, each line's data read once per pass.
  double own0 = 0.0, own2 = 0.0, own4 = 0.0;
  if constexpr (!STRUCT) {
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      own0 += h_flow_p(r.s, r.G, r.w7, r.fr ? 5 : 9);
      own2 += h_flow_p(r.s, r.G, r.w7, r.fr ? 7 : 11);
      own4 += h_flow_p(r.s, r.G, r.w7, r.fr ? 12 : 14);
    }
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      own0 += h_flow_q(r.s, r.B, r.w8, r.fr ? 5 : 9);
      own2 += h_flow_q(r.s, r.B, r.w8, r.fr ? 7 : 11);
      own4 += h_flow_q(r.s, r.B, r.w8, r.fr ? 12 : 14);
    }
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      const double jv_ = JP(r, false, false), jt_ = JP(r, false, true);
      own0 += pair_term(r.d7, jv_, jv_);
      own2 += pair_term(r.d7, jt_, jv_);
      own4 += pair_term(r.d7, jt_, jt_);
    }
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      const double jv_ = JQ(r, false, false), jt_ = JQ(r, false, true);
      own0 += pair_term(r.d8, jv_, jv_);
      own2 += pair_term(r.d8, jt_, jv_);
      own4 += pair_term(r.d8, jt_, jt_);
    }
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      own4 += pair_term(r.d10, r.fr ? 1.0 : -1.0, r.fr ? 1.0 : -1.0);
    }
    own0 += in.dw + sxv;
    own4 += in.dw + sxt;
  }
  for (int32_t q = p0; q < p1; ++q) {
    const unsigned long long code = code_next;
    if (q + 1 < p1) code_next = __ldg(t.bprog + q + 1);
    const uint32_t mask = (uint32_t)code;
    const int type = (int)((code >> 32) & 7);
    const int32_t rent = (int32_t)(code >> 35);
    double acc = 0.0;
    if constexpr (!STRUCT) {
      if (type == 0) {
        acc = own0;
      } else if (type == 2) {
        acc = own2;
      } else if (type == 4) {
        acc = own4;
      } else if ((mask & (mask - 1)) == 0) {  // one line to the neighbour: its terms in pass order
        const LV r = lv(__ffs(mask) - 1);
        if (type == 1) {  // (v_o, v_n), o > n
          acc += h_flow_p(r.s, r.G, r.w7, 6);
          acc += h_flow_q(r.s, r.B, r.w8, 6);
          acc += pair_term(r.d7, JP(r, true, false), JP(r, false, false));
          acc += pair_term(r.d8, JQ(r, true, false), JQ(r, false, false));
        } else if (type == 3) {  // (th_o, v_n)
          acc += h_flow_p(r.s, r.G, r.w7, r.fr ? 8 : 10);
          acc += h_flow_q(r.s, r.B, r.w8, r.fr ? 8 : 10);
          acc += pair_term(r.d7, JP(r, true, true), JP(r, false, false));
          acc += pair_term(r.d8, JQ(r, true, true), JQ(r, false, false));
        } else {  // (th_o, th_n), o > n
          acc += h_flow_p(r.s, r.G, r.w7, 13);
          acc += h_flow_q(r.s, r.B, r.w8, 13);
          acc += pair_term(r.d7, JP(r, true, true), JP(r, false, true));
          acc += pair_term(r.d8, JQ(r, true, true), JQ(r, false, true));
          acc += pair_term(r.d10, r.fr ? -1.0 : 1.0, r.fr ? 1.0 : -1.0);
        }
      } else {  // parallel lines: pass-major over the group
        switch (type) {
          case 1:  // (v_o, v_n), o > n
            PASS(h_flow_p(r.s, r.G, w7(r), 6));
            PASS(h_flow_q(r.s, r.B, w8(r), 6));
            PASS(pair_term(d7(r), JP(r, true, false), JP(r, false, false)));
            PASS(pair_term(d8(r), JQ(r, true, false), JQ(r, false, false)));
            break;
          case 3:  // (th_o, v_n)
            PASS(h_flow_p(r.s, r.G, w7(r), r.fr ? 8 : 10));
            PASS(h_flow_q(r.s, r.B, w8(r), r.fr ? 8 : 10));
            PASS(pair_term(d7(r), JP(r, true, true), JP(r, false, false)));
            PASS(pair_term(d8(r), JQ(r, true, true), JQ(r, false, false)));
            break;
          default:  // (th_o, th_n), o > n
            PASS(h_flow_p(r.s, r.G, w7(r), 13));
            PASS(h_flow_q(r.s, r.B, w8(r), 13));
            PASS(pair_term(d7(r), JP(r, true, true), JP(r, false, true)));
            PASS(pair_term(d8(r), JQ(r, true, true), JQ(r, false, true)));
            PASS(pair_term(d10(r), r.fr ? -1.0 : 1.0, r.fr ? 1.0 : -1.0));
            break;
        }
      }
    }
    const bool in_v = type < 4;
    const int64_t at = in_v ? posv + jv : post + jt;
    if constexpr (STRUCT) rows[at] = col((type == 0 || type == 1) ? off_v : off_th, rent);
    else M[at] = acc;
    if (in_v) ++jv; else ++jt;
  }
#undef PASS
  if (STRUCT) {
    if (cv >= 0 && posv + jv != __ldg(t.colptr + cv + 1)) atomicOr(bad, 1);
    if (ct >= 0 && post + jt != __ldg(t.colptr + ct + 1)) atomicOr(bad, 1);
  }
}

// Cooperative value pass of the slot-program class (GN_BUS3_COOP): one CTA of kB3C warps per
// (bus, 32 periods) instead of one warp.  The bus's line states are computed by the warps in
// parallel (line i by warp i mod kB3C) into the CTA's shared memory; after one barrier warp 0
// runs the fused own-slot sweep and writes the three own slots while the other warps take
// the neighbour slots round-robin.  Every slot keeps its summation order (each value is still
// one thread's ordered sum), so M is bit-identical to k_fz_bus3.  These buses are few (degree
// 8 and up, or parallel lines: ~0.3-1.5% of them) and sit at the end of the bus lane, where
// their one-warp latency chains were ~20 us.
#ifndef GN_BUS3_COOP
#define GN_BUS3_COOP 1
#endif
constexpr int kB3C = 4;
__global__ void __launch_bounds__(kB3C * 32) k_fz_bus3c(OpfKktTab t, const int4* __restrict__ buses,
                                                        int32_t n_buses, int32_t maxdeg, FIn in,
                                                        const double* __restrict__ dv,
                                                        double* __restrict__ M) {
  extern __shared__ double bsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n64 = blockIdx.x / t.tchunks;
  if (n64 >= n_buses) return;  // block-uniform
  const int4 bd0 = __ldg(buses + kBusDesc * n64), bd1 = __ldg(buses + kBusDesc * n64 + 1);
  const int4 bd2 = __ldg(buses + kBusDesc * n64 + 2);
  const int32_t n = bd0.x, b0 = bd0.y, deg = bd0.z & 255, T = t.T;
  const int32_t tt = (int32_t)(blockIdx.x - n64 * t.tchunks) * 32 + lane;
  const bool live = tt < T;
  const int32_t ts = live ? tt : T - 1;  // idle lanes load a valid period, write nothing
  double* S = bsm + lane;  // [line][field][lane]
  struct LU {
    double G, B;
    int32_t l, fr;
  };
  LU* U = reinterpret_cast<LU*>(bsm + (size_t)maxdeg * kSV * 32);
  if (threadIdx.x < deg) {
    const int2 e = __ldg(t.blx + b0 + threadIdx.x);
    const double2 gb = __ldg(t.blgb + b0 + threadIdx.x);
    U[threadIdx.x] = LU{gb.x, gb.y, e.x >> 1, e.x & 1};
  }
  for (int i = warp; i < deg; i += kB3C) {  // phase 1: line states, in parallel over warps
    const int2 e = __ldg(t.blx + b0 + i);
    const double2 gb = __ldg(t.blgb + b0 + i);
    const int32_t l = e.x >> 1, f = (e.x & 1) ? n : e.y, to = (e.x & 1) ? e.y : n;
    const int32_t rl = l * T + ts;
    const LineState st = line_state(gb.x, gb.y, in.x[t.v0 + f * T + ts], in.x[t.v0 + to * T + ts],
                                    in.x[t.th0 + f * T + ts], in.x[t.th0 + to * T + ts]);
    double* q = S + (size_t)i * kSV * 32;
    q[0 * 32] = st.Cs;
    q[1 * 32] = st.Sn;
    q[2 * 32] = st.cs;
    q[3 * 32] = st.sn;
    q[4 * 32] = st.vf;
    q[5 * 32] = st.vt;
    q[6 * 32] = in.w[t.flow_p0 + rl];
    q[7 * 32] = in.w[t.flow_q0 + rl];
    q[8 * 32] = dval(t, dv, t.flow_p0 + rl);
    q[9 * 32] = dval(t, dv, t.flow_q0 + rl);
    q[10 * 32] = dval(t, dv, t.ang0 + rl);
  }
  __syncthreads();
  struct LV {
    LineState s;
    double G, B;
    double w7, w8, d7, d8, d10;
    int32_t l, fr;
  };
  auto lv = [&](int k) {
    LV r;
    const LU u = U[k];
    r.l = u.l;
    r.fr = u.fr;
    r.G = u.G;
    r.B = u.B;
    const double* q = S + (size_t)k * kSV * 32;
    r.s.Cs = q[0 * 32];
    r.s.Sn = q[1 * 32];
    r.s.cs = q[2 * 32];
    r.s.sn = q[3 * 32];
    r.s.vf = q[4 * 32];
    r.s.vt = q[5 * 32];
    r.s.vfvt = r.s.vf * r.s.vt;
    r.w7 = q[6 * 32];
    r.w8 = q[7 * 32];
    r.d7 = q[8 * 32];
    r.d8 = q[9 * 32];
    r.d10 = q[10 * 32];
    return r;
  };
  auto JP = [&](const LV& r, bool other, bool theta) {
    const int f = theta ? ((r.fr ^ other) ? 3 : 4) : ((r.fr ^ other) ? 1 : 2);
    return j_flow_p(r.s, r.G, r.B, f);
  };
  auto JQ = [&](const LV& r, bool other, bool theta) {
    const int f = theta ? ((r.fr ^ other) ? 3 : 4) : ((r.fr ^ other) ? 1 : 2);
    return j_flow_q(r.s, r.G, r.B, f);
  };
  const int32_t cv = bd1.x < 0 ? -1 : bd1.x * T + ts, ct = bd1.y < 0 ? -1 : bd1.y * T + ts;
  const int64_t posv = cv >= 0 ? (int64_t)bd2.x + (int64_t)ts * bd2.y : 0;
  const int64_t post = ct >= 0 ? (int64_t)bd2.z + (int64_t)ts * bd2.w : 0;
  const int32_t p0 = bd0.w, p1 = p0 + (bd0.z >> 8);
  double own0 = 0.0, own2 = 0.0, own4 = 0.0;
  if (warp == 0) {  // the own slots: one fused pass-major sweep over every incident line
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      own0 += h_flow_p(r.s, r.G, r.w7, r.fr ? 5 : 9);
      own2 += h_flow_p(r.s, r.G, r.w7, r.fr ? 7 : 11);
      own4 += h_flow_p(r.s, r.G, r.w7, r.fr ? 12 : 14);
    }
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      own0 += h_flow_q(r.s, r.B, r.w8, r.fr ? 5 : 9);
      own2 += h_flow_q(r.s, r.B, r.w8, r.fr ? 7 : 11);
      own4 += h_flow_q(r.s, r.B, r.w8, r.fr ? 12 : 14);
    }
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      const double jv_ = JP(r, false, false), jt_ = JP(r, false, true);
      own0 += pair_term(r.d7, jv_, jv_);
      own2 += pair_term(r.d7, jt_, jv_);
      own4 += pair_term(r.d7, jt_, jt_);
    }
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      const double jv_ = JQ(r, false, false), jt_ = JQ(r, false, true);
      own0 += pair_term(r.d8, jv_, jv_);
      own2 += pair_term(r.d8, jt_, jv_);
      own4 += pair_term(r.d8, jt_, jt_);
    }
    for (int k = 0; k < deg; ++k) {
      const LV r = lv(k);
      own4 += pair_term(r.d10, r.fr ? 1.0 : -1.0, r.fr ? 1.0 : -1.0);
    }
    own0 += in.dw + (cv >= 0 ? in.sx[cv] : 0.0);
    own4 += in.dw + (ct >= 0 ? in.sx[ct] : 0.0);
  }
#define PASS(expr)                                 \
  for (uint32_t mm = mask; mm; mm &= mm - 1) {     \
    const LV r = lv(__ffs(mm) - 1);                \
    acc += (expr);                                 \
  }
  int jv = 0, jt = 0, nb = 0;
  for (int32_t q = p0; q < p1; ++q) {  // every warp walks the program (slot positions)
    const unsigned long long code = __ldg(t.bprog + q);
    const uint32_t mask = (uint32_t)code;
    const int type = (int)((code >> 32) & 7);
    const bool in_v = type < 4;
    const int64_t at = in_v ? posv + jv : post + jt;
    if (in_v) ++jv; else ++jt;
    const bool own = type == 0 || type == 2 || type == 4;
    const int owner = own ? 0 : 1 + (nb++ % (kB3C - 1));
    if (owner != warp) continue;
    double acc = 0.0;
    if (own) {
      acc = type == 0 ? own0 : (type == 2 ? own2 : own4);
    } else if ((mask & (mask - 1)) == 0) {  // one line to the neighbour: its terms in pass order
      const LV r = lv(__ffs(mask) - 1);
      if (type == 1) {
        acc += h_flow_p(r.s, r.G, r.w7, 6);
        acc += h_flow_q(r.s, r.B, r.w8, 6);
        acc += pair_term(r.d7, JP(r, true, false), JP(r, false, false));
        acc += pair_term(r.d8, JQ(r, true, false), JQ(r, false, false));
      } else if (type == 3) {
        acc += h_flow_p(r.s, r.G, r.w7, r.fr ? 8 : 10);
        acc += h_flow_q(r.s, r.B, r.w8, r.fr ? 8 : 10);
        acc += pair_term(r.d7, JP(r, true, true), JP(r, false, false));
        acc += pair_term(r.d8, JQ(r, true, true), JQ(r, false, false));
      } else {
        acc += h_flow_p(r.s, r.G, r.w7, 13);
        acc += h_flow_q(r.s, r.B, r.w8, 13);
        acc += pair_term(r.d7, JP(r, true, true), JP(r, false, true));
        acc += pair_term(r.d8, JQ(r, true, true), JQ(r, false, true));
        acc += pair_term(r.d10, r.fr ? -1.0 : 1.0, r.fr ? 1.0 : -1.0);
      }
    } else {  // parallel lines: pass-major over the group
      switch (type) {
        case 1:
          PASS(h_flow_p(r.s, r.G, r.w7, 6));
          PASS(h_flow_q(r.s, r.B, r.w8, 6));
          PASS(pair_term(r.d7, JP(r, true, false), JP(r, false, false)));
          PASS(pair_term(r.d8, JQ(r, true, false), JQ(r, false, false)));
          break;
        case 3:
          PASS(h_flow_p(r.s, r.G, r.w7, r.fr ? 8 : 10));
          PASS(h_flow_q(r.s, r.B, r.w8, r.fr ? 8 : 10));
          PASS(pair_term(r.d7, JP(r, true, true), JP(r, false, false)));
          PASS(pair_term(r.d8, JQ(r, true, true), JQ(r, false, false)));
          break;
        default:
          PASS(h_flow_p(r.s, r.G, r.w7, 13));
          PASS(h_flow_q(r.s, r.B, r.w8, 13));
          PASS(pair_term(r.d7, JP(r, true, true), JP(r, false, true)));
          PASS(pair_term(r.d8, JQ(r, true, true), JQ(r, false, true)));
          PASS(pair_term(r.d10, r.fr ? -1.0 : 1.0, r.fr ? 1.0 : -1.0));
          break;
      }
    }
    if (live && (in_v ? cv >= 0 : ct >= 0)) M[at] = acc;
  }
#undef PASS
}

// Register-resident variant for buses of exactly DEG lines and no parallel lines
// (almost every bus of a transmission network): each lane holds its period's
// state and row inputs of all DEG lines in registers; the own slots are one
// pass-major sweep, each neighbour slot is its line's terms in pass order, and
// every value goes to its precomputed offset in the column (bpos, boff).
template <int DEG, bool STRUCT>
__device__ __forceinline__ void busr_body(int64_t vblock, const OpfKktTab& t,
                                          const int4* __restrict__ buses, int32_t n_buses,
                                          const FIn& in, const double* __restrict__ dv,
                                          double* __restrict__ M, int32_t* __restrict__ rows,
                                          int32_t* __restrict__ bad) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = vblock * kBW3 + warp;
  const int32_t T = t.T;
#if GN_BUSR_FLAT
  // flat (bus, period) items: lane i of warp w takes item 32 w + i, so no lane idles when T
  // is not a multiple of 32 (a period shard of 21, configs[1]'s 24, configs[2]'s 48)
  const int64_t item = w * 32 + lane;
  const int64_t n64 = item / T;
  if (n64 >= n_buses) return;
  const int32_t tt = (int32_t)(item - n64 * T);
#else
  const int64_t n64 = w / t.tchunks;
  if (n64 >= n_buses) return;
  const int32_t tt = (int32_t)(w - n64 * t.tchunks) * 32 + lane;
  if (tt >= T) return;
#endif
  const int4* bd = buses + (int64_t)bus_desc_stride(DEG - 1) * n64;
  const int4 bd0 = __ldg(bd), bd1 = __ldg(bd + 1), bd2 = __ldg(bd + 2);
  int2 e[DEG];
  int32_t pp[DEG];
  double2 gb[DEG];
#pragma unroll
  for (int i = 0; i < DEG; ++i) {  // the lines inline in the descriptor: no dependent level
    const int4 q = __ldg(bd + kBusDesc + i);
    e[i] = make_int2(q.x, q.y);
    pp[i] = q.z;
    const int4 g = __ldg(bd + kBusDesc + DEG + i);
    gb[i] = make_double2(__hiloint2double(g.y, g.x), __hiloint2double(g.w, g.z));
  }
  const int32_t n = bd0.x, boff = bd0.w;
  const int32_t cv = bd1.x < 0 ? -1 : bd1.x * T + tt, ct = bd1.y < 0 ? -1 : bd1.y * T + tt;
  const int64_t posv = cv >= 0 ? (int64_t)bd2.x + (int64_t)tt * bd2.y : 0;
  const int64_t post = ct >= 0 ? (int64_t)bd2.z + (int64_t)tt * bd2.w : 0;
  if constexpr (STRUCT) {
    const int32_t off_v = 2 * t.G + 2 * t.L, off_th = off_v + t.N;
    auto col = [&](int32_t off, int32_t ent) {
      const int32_t k = __ldg(t.lent + off + ent);
      return k < 0 ? -1 : k * T + tt;
    };
    int32_t nv = 0, nt_ = 0;
    if (cv >= 0) {
      rows[posv] = cv;
      ++nv;
      if (ct >= 0) {
        rows[posv + boff] = ct;
        ++nv;
      }
    }
    if (ct >= 0) {
      rows[post] = ct;
      ++nt_;
    }
#pragma unroll
    for (int i = 0; i < DEG; ++i) {
      const int32_t o = e[i].y, p1 = pp[i] & 0xff, p3 = (pp[i] >> 8) & 0xff, p5 = (pp[i] >> 16) & 0xff;
      if (p1 != 0xff && cv >= 0) { rows[posv + p1] = col(off_v, o); ++nv; }
      if (p3 != 0xff && cv >= 0) { rows[posv + p3] = col(off_th, o); ++nv; }
      if (p5 != 0xff && ct >= 0) { rows[post + p5] = col(off_th, o); ++nt_; }
    }
    if ((cv >= 0 && posv + nv != __ldg(t.colptr + cv + 1)) ||
        (ct >= 0 && post + nt_ != __ldg(t.colptr + ct + 1)) || (cv >= 0 && ct >= 0 && boff < 0))
      atomicOr(bad, 1);
    return;
  }
  // ---- loads (all independent), then the line states
  double xvf[DEG], xvt[DEG], xtf[DEG], xtt[DEG], w7[DEG], w8[DEG], d7[DEG], d8[DEG], d10[DEG];
#pragma unroll
  for (int i = 0; i < DEG; ++i) {
    const bool fr = e[i].x & 1;
    const int32_t l = e[i].x >> 1, o = e[i].y, f = fr ? n : o, to = fr ? o : n;
    const int32_t rl = l * T + tt;
    xvf[i] = in.x[t.v0 + f * T + tt];
    xvt[i] = in.x[t.v0 + to * T + tt];
    xtf[i] = in.x[t.th0 + f * T + tt];
    xtt[i] = in.x[t.th0 + to * T + tt];
    w7[i] = in.w[t.flow_p0 + rl];
    w8[i] = in.w[t.flow_q0 + rl];
    d7[i] = dval(t, dv, t.flow_p0 + rl);
    d8[i] = dval(t, dv, t.flow_q0 + rl);
    d10[i] = dval(t, dv, t.ang0 + rl);
  }
  const double sxv = cv >= 0 ? in.sx[cv] : 0.0, sxt = ct >= 0 ? in.sx[ct] : 0.0;
  LineState st[DEG];
#pragma unroll
  for (int i = 0; i < DEG; ++i) st[i] = line_state(gb[i].x, gb[i].y, xvf[i], xvt[i], xtf[i], xtt[i]);
  // own slots, pass-major over the lines (ascending l)
  double own0 = 0.0, own2 = 0.0, own4 = 0.0;
#pragma unroll
  for (int i = 0; i < DEG; ++i) {
    const bool fr = e[i].x & 1;
    own0 += h_flow_p(st[i], gb[i].x, w7[i], fr ? 5 : 9);
    own2 += h_flow_p(st[i], gb[i].x, w7[i], fr ? 7 : 11);
    own4 += h_flow_p(st[i], gb[i].x, w7[i], fr ? 12 : 14);
  }
#pragma unroll
  for (int i = 0; i < DEG; ++i) {
    const bool fr = e[i].x & 1;
    own0 += h_flow_q(st[i], gb[i].y, w8[i], fr ? 5 : 9);
    own2 += h_flow_q(st[i], gb[i].y, w8[i], fr ? 7 : 11);
    own4 += h_flow_q(st[i], gb[i].y, w8[i], fr ? 12 : 14);
  }
#pragma unroll
  for (int i = 0; i < DEG; ++i) {
    const bool fr = e[i].x & 1;
    const double jv = j_flow_p(st[i], gb[i].x, gb[i].y, fr ? 1 : 2);
    const double jt = j_flow_p(st[i], gb[i].x, gb[i].y, fr ? 3 : 4);
    own0 += pair_term(d7[i], jv, jv);
    own2 += pair_term(d7[i], jt, jv);
    own4 += pair_term(d7[i], jt, jt);
  }
#pragma unroll
  for (int i = 0; i < DEG; ++i) {
    const bool fr = e[i].x & 1;
    const double jv = j_flow_q(st[i], gb[i].x, gb[i].y, fr ? 1 : 2);
    const double jt = j_flow_q(st[i], gb[i].x, gb[i].y, fr ? 3 : 4);
    own0 += pair_term(d8[i], jv, jv);
    own2 += pair_term(d8[i], jt, jv);
    own4 += pair_term(d8[i], jt, jt);
  }
#pragma unroll
  for (int i = 0; i < DEG; ++i) {
    const bool fr = e[i].x & 1;
    own4 += pair_term(d10[i], fr ? 1.0 : -1.0, fr ? 1.0 : -1.0);
  }
  own0 += in.dw + sxv;
  own4 += in.dw + sxt;
  if (cv >= 0) {
    M[posv] = own0;
    if (ct >= 0) M[posv + boff] = own2;
  }
  if (ct >= 0) M[post] = own4;
  // neighbour slots: one line each, its terms in pass order
#pragma unroll
  for (int i = 0; i < DEG; ++i) {
    const bool fr = e[i].x & 1;
    const double G = gb[i].x, B = gb[i].y;
    const LineState& s = st[i];
    const int fvn = fr ? 1 : 2, fvo = fr ? 2 : 1, ftn = fr ? 3 : 4, fto = fr ? 4 : 3;
    const int32_t p1 = pp[i] & 0xff, p3 = (pp[i] >> 8) & 0xff, p5 = (pp[i] >> 16) & 0xff;
    if (p1 != 0xff && cv >= 0) {  // (v(o), v(n)), o > n
      double acc = 0.0;
      acc += h_flow_p(s, G, w7[i], 6);
      acc += h_flow_q(s, B, w8[i], 6);
      acc += pair_term(d7[i], j_flow_p(s, G, B, fvo), j_flow_p(s, G, B, fvn));
      acc += pair_term(d8[i], j_flow_q(s, G, B, fvo), j_flow_q(s, G, B, fvn));
      M[posv + p1] = acc;
    }
    if (p3 != 0xff && cv >= 0) {  // (th(o), v(n))
      double acc = 0.0;
      acc += h_flow_p(s, G, w7[i], fr ? 8 : 10);
      acc += h_flow_q(s, B, w8[i], fr ? 8 : 10);
      acc += pair_term(d7[i], j_flow_p(s, G, B, fto), j_flow_p(s, G, B, fvn));
      acc += pair_term(d8[i], j_flow_q(s, G, B, fto), j_flow_q(s, G, B, fvn));
      M[posv + p3] = acc;
    }
    if (p5 != 0xff && ct >= 0) {  // (th(o), th(n)), o > n
      double acc = 0.0;
      acc += h_flow_p(s, G, w7[i], 13);
      acc += h_flow_q(s, B, w8[i], 13);
      acc += pair_term(d7[i], j_flow_p(s, G, B, fto), j_flow_p(s, G, B, ftn));
      acc += pair_term(d8[i], j_flow_q(s, G, B, fto), j_flow_q(s, G, B, ftn));
      acc += pair_term(d10[i], fr ? -1.0 : 1.0, fr ? 1.0 : -1.0);
      M[post + p5] = acc;
    }
  }
}

template <int DEG, bool STRUCT>
__global__ void __launch_bounds__(kBW3 * 32, kBusrMinBlocks[DEG]) k_fz_busr(OpfKktTab t, int64_t nvb,
                                                    const int4* __restrict__ buses,
                                                    int32_t n_buses, FIn in,
                                                    const double* __restrict__ dv,
                                                    double* __restrict__ M,
                                                    int32_t* __restrict__ rows,
                                                    int32_t* __restrict__ bad) {
  if (nvb <= gridDim.x) {  // (uncapped grid: one virtual CTA per CTA)
    busr_body<DEG, STRUCT>(blockIdx.x, t, buses, n_buses, in, dv, M, rows, bad);
    return;
  }
  for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x)
    busr_body<DEG, STRUCT>(vb, t, buses, n_buses, in, dv, M, rows, bad);
}

template <int DEG>
static void launch_busr(const OpfKktTab& t, const int4* buses, int32_t n_buses, const FIn& in,
                        const double* dv, double* M, int32_t* rows, int32_t* bad, cudaStream_t s) {
  static const char* names[] = {"", "k_fz_busr<d1>", "k_fz_busr<d2>", "k_fz_busr<d3>",
                                "k_fz_busr<d4>", "k_fz_busr<d5>", "k_fz_busr<d6>",
                                "k_fz_busr<d7>", "k_fz_busr<d8>", "k_fz_busr<d9>"};
#if GN_BUSR_FLAT
  const int64_t warps = ((int64_t)n_buses * t.T + 31) / 32;
#else
  const int64_t warps = (int64_t)n_buses * t.tchunks;
#endif
  const int64_t nvb = (warps + kBW3 - 1) / kBW3;
  KTimer kt(names[DEG], s);
  if (rows)
    k_fz_busr<DEG, true><<<grid_cap(nvb, t.grid_cap * GN_BUSR_CAP_MUL), kBW3 * 32, 0, s>>>(t, nvb, buses, n_buses, in, dv, M,
                                                             rows, bad);
  else
    k_fz_busr<DEG, false><<<grid_cap(nvb, t.grid_cap * GN_BUSR_CAP_MUL), kBW3 * 32, 0, s>>>(t, nvb, buses, n_buses, in, dv, M,
                                                              rows, bad);
  count_launch();
}

bool fz_bus_fits(int32_t maxdeg) {
  const size_t md = maxdeg > 0 ? maxdeg : 1;
  return maxdeg <= 32 && md * (kSV * 32 * sizeof(double) + 24) <= kBusSmemMax;
}

void launch_fz_bus(const OpfKktTab& t, const int4* buses, int32_t n_buses, int32_t maxdeg,
                   int klass, const FIn& in, const double* dv, double* M, int32_t* rows, int32_t* bad,
                   cudaStream_t s) {
  if (n_buses <= 0) return;
  if (klass < kBusRegMax) {
    switch (klass) {
      case 0: return launch_busr<1>(t, buses, n_buses, in, dv, M, rows, bad, s);
      case 1: return launch_busr<2>(t, buses, n_buses, in, dv, M, rows, bad, s);
      case 2: return launch_busr<3>(t, buses, n_buses, in, dv, M, rows, bad, s);
      case 3: return launch_busr<4>(t, buses, n_buses, in, dv, M, rows, bad, s);
      case 4: return launch_busr<5>(t, buses, n_buses, in, dv, M, rows, bad, s);
      case 5: return launch_busr<6>(t, buses, n_buses, in, dv, M, rows, bad, s);
      case 6: if constexpr (kBusRegMax > 6) return launch_busr<7>(t, buses, n_buses, in, dv, M, rows, bad, s);
              break;
      case 7: if constexpr (kBusRegMax > 7) return launch_busr<8>(t, buses, n_buses, in, dv, M, rows, bad, s);
              break;
      case 8: if constexpr (kBusRegMax > 8) return launch_busr<9>(t, buses, n_buses, in, dv, M, rows, bad, s);
              break;
      default: break;
    }
  }
  const int64_t warps = (int64_t)n_buses * t.tchunks;
  const int md = maxdeg > 0 ? maxdeg : 1;
  int nw = kBW3;
  while (nw > 1 && (size_t)nw * md * (kSV * 32 * sizeof(double) + 24) > kBusSmemMax) nw >>= 1;
  const size_t smem = (size_t)nw * md * (kSV * 32 * sizeof(double) + 24);
  if (smem > kBusSmemMax) throw Error(GN_ERR_UNSUPPORTED, "bus degree too large for the fused kernel");
  const unsigned blocks = (unsigned)((warps + nw - 1) / nw);
  {  // the dynamic shared-memory opt-in is per device (contexts on several GPUs)
    static std::mutex mu;
    static std::vector<char> done;
    int dev = 0;
    GN_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (static_cast<size_t>(dev) >= done.size()) done.resize(static_cast<size_t>(dev) + 1, 0);
    if (!done[dev]) {
      GN_CK(cudaFuncSetAttribute(k_fz_bus3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kBusSmemMax));
      GN_CK(cudaFuncSetAttribute(k_fz_bus3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kBusSmemMax));
      done[dev] = 1;
    }
  }
  KTimer kt(klass == kBusRegMax ? "k_fz_bus3<le8>" : "k_fz_bus3<rest>", s);
#if GN_BUS3_COOP
  if (!rows) {
    const size_t csmem = (size_t)md * (kSV * 32 * sizeof(double) + 24);
    static std::mutex cmu;
    static std::vector<char> cdone;
    int dev = 0;
    GN_CK(cudaGetDevice(&dev));
    {
      std::lock_guard<std::mutex> lock(cmu);
      if (static_cast<size_t>(dev) >= cdone.size()) cdone.resize(static_cast<size_t>(dev) + 1, 0);
      if (!cdone[dev]) {
        GN_CK(cudaFuncSetAttribute(k_fz_bus3c, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kBusSmemMax));
        cdone[dev] = 1;
      }
    }
    k_fz_bus3c<<<(unsigned)((int64_t)n_buses * t.tchunks), kB3C * 32, csmem, s>>>(
        t, buses, n_buses, md, in, dv, M);
    count_launch();
    return;
  }
#endif
  if (rows)
    k_fz_bus3<true><<<blocks, nw * 32, smem, s>>>(t, buses, n_buses, md, in, dv, M, rows, bad);
  else
    k_fz_bus3<false><<<blocks, nw * 32, smem, s>>>(t, buses, n_buses, md, in, dv, M, rows, bad);
  count_launch();
}

}  // namespace gnb
