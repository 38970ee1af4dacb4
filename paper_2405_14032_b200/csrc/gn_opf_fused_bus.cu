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
#include "gn_opf_kkt.cuh"
#include "gn_opf_math.cuh"

namespace gnb {

constexpr int kBW2 = 4;  // warps per CTA

// terms of one (line, bus side, period)
struct BusTerms {
  double hv7, hv8, pv7, pv8;           // (v_n, v_n)
  double hs7, hs8, ps7, ps8;           // (th_n, v_n)
  double ht7, ht8, pt7, pt8, pt10;     // (th_n, th_n)
  double ho7, ho8, po7, po8;           // (v_o, v_n), o > n
  double hx7, hx8, px7, px8;           // (th_o, v_n)
  double hy7, hy8, py7, py8, py10;     // (th_o, th_n), o > n
};

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

template <bool STRUCT>
__global__ void __launch_bounds__(kBW2 * 32) k_fz_bus2(OpfKktTab t, const int2* __restrict__ items,
                                                       int64_t n_items, FIn in,
                                                       const double* __restrict__ dv,
                                                       double* __restrict__ M,
                                                       int32_t* __restrict__ rows,
                                                       int32_t* __restrict__ bad) {
  const int64_t w = ((int64_t)blockIdx.x * kBW2 * 32 + threadIdx.x) >> 5;
  if (w >= n_items) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int2 it = items[w];
  const int32_t n = it.x, T = t.T;
  const int32_t b0 = __ldg(t.bl_ptr + n), deg = __ldg(t.bl_ptr + n + 1) - b0;
  int P = 1;
  while (P < deg) P <<= 1;
  const int g = lane / P, i = lane - g * P;
  const int base = g * P;  // lane of line slot 0 of this period group
  const int32_t tt = it.y + g;
  const bool tvalid = (g < 32 / P) && tt < T;
  const bool writer = tvalid && i == 0;
  const int32_t tc = tvalid ? tt : 0;  // safe period for idle lanes
  const int32_t off_v = 2 * t.G + 2 * t.L, off_th = off_v + t.N;

  // ---------------------------------------------------------------- terms
  BusTerms b{};
  if constexpr (!STRUCT) {
    if (i < deg) {
      const int32_t e = __ldg(t.bl + b0 + i), l = e >> 1, fr = e & 1;
      const int32_t f = __ldg(t.lf + l), to = __ldg(t.lt + l);
      const double G = __ldg(t.lg + l), B = __ldg(t.lb + l);
      const int64_t lt_ = (int64_t)l * T + tc;
      const LineState s =
          line_state(G, B, in.x[t.v0 + (int64_t)f * T + tc], in.x[t.v0 + (int64_t)to * T + tc],
                     in.x[t.th0 + (int64_t)f * T + tc], in.x[t.th0 + (int64_t)to * T + tc]);
      const double w7 = in.w[t.flow_p0 + lt_], w8 = in.w[t.flow_q0 + lt_];
      const double d7 = dv[t.flow_p0 + lt_], d8 = dv[t.flow_q0 + lt_], d10 = dv[t.ang0 + lt_];
      const int vn = fr ? 1 : 2, vo = fr ? 2 : 1, tn = fr ? 3 : 4, to4 = fr ? 4 : 3;
      const double p_vn = j_flow_p(s, G, B, vn), p_vo = j_flow_p(s, G, B, vo);
      const double p_tn = j_flow_p(s, G, B, tn), p_to = j_flow_p(s, G, B, to4);
      const double q_vn = j_flow_q(s, G, B, vn), q_vo = j_flow_q(s, G, B, vo);
      const double q_tn = j_flow_q(s, G, B, tn), q_to = j_flow_q(s, G, B, to4);
      const double an = fr ? 1.0 : -1.0, ao = -an;
      b.hv7 = h_flow_p(s, G, w7, fr ? 5 : 9);
      b.hv8 = h_flow_q(s, B, w8, fr ? 5 : 9);
      b.pv7 = pair_term(d7, p_vn, p_vn);
      b.pv8 = pair_term(d8, q_vn, q_vn);
      b.hs7 = h_flow_p(s, G, w7, fr ? 7 : 11);
      b.hs8 = h_flow_q(s, B, w8, fr ? 7 : 11);
      b.ps7 = pair_term(d7, p_tn, p_vn);
      b.ps8 = pair_term(d8, q_tn, q_vn);
      b.ht7 = h_flow_p(s, G, w7, fr ? 12 : 14);
      b.ht8 = h_flow_q(s, B, w8, fr ? 12 : 14);
      b.pt7 = pair_term(d7, p_tn, p_tn);
      b.pt8 = pair_term(d8, q_tn, q_tn);
      b.pt10 = pair_term(d10, an, an);
      b.ho7 = h_flow_p(s, G, w7, 6);
      b.ho8 = h_flow_q(s, B, w8, 6);
      b.po7 = pair_term(d7, p_vo, p_vn);
      b.po8 = pair_term(d8, q_vo, q_vn);
      b.hx7 = h_flow_p(s, G, w7, fr ? 8 : 10);
      b.hx8 = h_flow_q(s, B, w8, fr ? 8 : 10);
      b.px7 = pair_term(d7, p_to, p_vn);
      b.px8 = pair_term(d8, q_to, q_vn);
      b.hy7 = h_flow_p(s, G, w7, 13);
      b.hy8 = h_flow_q(s, B, w8, 13);
      b.py7 = pair_term(d7, p_to, p_tn);
      b.py8 = pair_term(d8, q_to, q_tn);
      b.py10 = pair_term(d10, ao, an);
    }
  }
  // Per-bus slot program (built on the host, opf_kkt_prepare): each slot is
  // (lane mask of its lines, type, row entity); types 0-3 belong to v(n),
  // 4-5 to th(n).  Mask bits ascend with l, so the shuffle order is the
  // reference's record order.
  const int32_t p0 = __ldg(t.bprog_ptr + n), p1 = __ldg(t.bprog_ptr + n + 1);
  auto col = [&](int32_t off, int32_t e) {
    const int32_t k = __ldg(t.lent + off + e);
    return k < 0 ? -1 : k * T + tc;
  };
  const int32_t cv = col(off_v, n), ct = col(off_th, n);
  const int64_t posv = cv >= 0 ? (int64_t)__ldg(t.colptr + cv) : 0;
  const int64_t post = ct >= 0 ? (int64_t)__ldg(t.colptr + ct) : 0;
  int jv = 0, jt = 0;
#define MSUM(fld)                                                     \
  for (uint32_t mm = mask; mm; mm &= mm - 1) acc += shfl(b.fld, base + __ffs(mm) - 1)
  for (int32_t q = p0; q < p1; ++q) {
    const unsigned long long code = __ldg(t.bprog + q);
    const uint32_t mask = (uint32_t)code;
    const int type = (int)((code >> 32) & 7);
    const int32_t rent = (int32_t)(code >> 35);
    double acc = 0.0;
    switch (type) {
      case 0: MSUM(hv7); MSUM(hv8); MSUM(pv7); MSUM(pv8); break;
      case 1: MSUM(ho7); MSUM(ho8); MSUM(po7); MSUM(po8); break;
      case 2: MSUM(hs7); MSUM(hs8); MSUM(ps7); MSUM(ps8); break;
      case 3: MSUM(hx7); MSUM(hx8); MSUM(px7); MSUM(px8); break;
      case 4: MSUM(ht7); MSUM(ht8); MSUM(pt7); MSUM(pt8); MSUM(pt10); break;
      default: MSUM(hy7); MSUM(hy8); MSUM(py7); MSUM(py8); MSUM(py10); break;
    }
    const bool in_v = type < 4;
    if (writer) {
      const int32_t cc = in_v ? cv : ct;
      if (type == 0 || type == 4) acc += in.dw + in.sx[cc];  // diagonal
      const int64_t at = in_v ? posv + jv : post + jt;
      if constexpr (STRUCT) {
        const int32_t row = col((type == 1 || type == 0) ? off_v : off_th, rent);
        rows[at] = row;
      } else {
        M[at] = acc;
      }
    }
    if (in_v) ++jv; else ++jt;
  }
#undef MSUM
  if (STRUCT && writer) {
    if (cv >= 0 && posv + jv != __ldg(t.colptr + cv + 1)) atomicOr(bad, 1);
    if (ct >= 0 && post + jt != __ldg(t.colptr + ct + 1)) atomicOr(bad, 1);
  }
}

void launch_fz_bus(const OpfKktTab& t, const int2* items, int64_t n_items, const FIn& in,
                   const double* dv, double* M, int32_t* rows, int32_t* bad, cudaStream_t s) {
  const unsigned blocks = (unsigned)((n_items + kBW2 - 1) / kBW2);
  if (rows)
    k_fz_bus2<true><<<blocks, kBW2 * 32, 0, s>>>(t, items, n_items, in, dv, M, rows, bad);
  else
    k_fz_bus2<false><<<blocks, kBW2 * 32, 0, s>>>(t, items, n_items, in, dv, M, rows, bad);
  count_launch();
}

}  // namespace gnb
