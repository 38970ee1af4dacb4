// Per-element NLP callbacks: one block body per element class (line x period
// with its rated-line thermal rows, generator x period, ramping-generator x step,
// bus x period), each writing its patterns' COO slots in the reference's
// freeze order.  Each callback is ONE launch (k_eval<MODE>) whose grid is the
// concatenation of the classes' block ranges (heavy line blocks first, the short
// generator / ramp blocks fill the tail), so a callback costs one kernel boundary.
// Closed-form derivatives of the 12 OPF patterns
// replace the reference's interpreted tape AD
// (model/tape.hpp); value expressions keep the tape's operation order and
// the library is built with -fmad=false, so g and J agree with the reference
// to the last bit except where CUDA's sin/cos differ from glibc's by an ulp.
//
//   evaluate_objective   pattern_model.hpp:278-300
//   evaluate_constraints pattern_model.hpp:302-326
//   evaluate_gradient    pattern_model.hpp:328-359
//   evaluate_jacobian    pattern_model.hpp:361-388
//   evaluate_hessian     pattern_model.hpp:393-436 (w == 0 -> zeros, :409-412)
#include "gn_eval.cuh"
#include "gn_opf_math.cuh"

namespace gnb {

// tuning-build switch (scripts/build_variant.py): balance-row blocks first in the trial launch
#ifndef GN_G_BUS_FIRST
#define GN_G_BUS_FIRST 1
#endif
#ifndef GN_EVAL_BS
#define GN_EVAL_BS 128
#endif
constexpr int kBS = GN_EVAL_BS;  // records per block (one per thread; 128 measured ahead of 256)

__device__ __forceinline__ void report(unsigned long long* st, int pid, int64_t rec) {
  atomicMin(st, (static_cast<unsigned long long>(pid) << 32) |
                    static_cast<unsigned long long>(rec));
}

// Block-cooperative contiguous store of `nb` records x K values staged in smem.
// The CTA's records occupy one contiguous span of the output; after the values are
// staged, one thread hands the span to the TMA bulk-copy engine
// (cp.async.bulk.global.shared::cta, SASS UBLKCP) instead of 15 rounds of per-thread
// stores.  The bulk copy needs 16-byte aligned source/destination and a multiple of
// 16 bytes: the staging is shifted by one double when the destination is 8 mod 16,
// and a leading / trailing odd element is stored directly.
template <int K>
__device__ __forceinline__ void stage_out(double* sm, const double (&v)[K], bool valid,
                                          double* __restrict__ out, int nb) {
  const int shift = (reinterpret_cast<uintptr_t>(out) & 15) ? 1 : 0;  // block-uniform
  if (valid) {
#pragma unroll
    for (int s = 0; s < K; ++s) sm[shift + threadIdx.x * K + s] = v[s];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> async proxy
  __syncthreads();
  if (threadIdx.x == 0) {
    const int total = nb * K;
    const int head = total > 0 ? shift : 0;
    if (head) out[0] = sm[shift];
    const int rest = total - head, body = rest & ~1;
    if (body > 0) {
      const unsigned src = static_cast<unsigned>(__cvta_generic_to_shared(sm + shift + head));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(out + head), "r"(src), "r"(body * 8) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (rest & 1) out[total - 1] = sm[shift + total - 1];
    // wait until the engine has READ the staging buffer (reusable, or the CTA may exit);
    // the global writes complete asynchronously, visible at the kernel boundary
    if (body > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncthreads();
}

// Contiguous region of nb records x K slots holding per-slot constants (K <= 3), written
// with 16-byte stores.  The constants are selected by constant indices (no local-memory
// table): the scalar, dynamically indexed version cost this region twice its bytes' time.
template <int K>
__device__ __forceinline__ double cpick(const double (&c)[K], int m) {
  static_assert(K >= 1 && K <= 3, "period");
  if constexpr (K == 1) return c[0];
  else if constexpr (K == 2) return m == 0 ? c[0] : c[1];
  else return m == 0 ? c[0] : (m == 1 ? c[1] : c[2]);
}
template <int K>
__device__ __forceinline__ void const_out(double* __restrict__ out, int nb,
                                          const double (&c)[K]) {
  const int total = nb * K;
  if (total <= 0) return;
  const int head = (reinterpret_cast<uintptr_t>(out) & 15) ? 1 : 0;  // to a 16-byte boundary
  if (head && threadIdx.x == 0) out[0] = c[0];
  const int rest = total - head, body = rest >> 1;
  double2* o2 = reinterpret_cast<double2*>(out + head);
  for (int j = threadIdx.x; j < body; j += kBS) {
    const int e = head + 2 * j;
    o2[j] = make_double2(cpick(c, e % K), cpick(c, (e + 1) % K));
  }
  if ((rest & 1) && threadIdx.x == 0) out[total - 1] = cpick(c, (total - 1) % K);
}

// ---------------------------------------------------------------- lines
// Patterns 1, 2 (balance-flow J/H), 7, 8 (flow definitions), 10 (angle), and
// 12 (thermal) for rated lines: its rows / records of (line k, period t) are
// written by the same thread, which already holds p and q.
template <int MODE>
__device__ __forceinline__ void line_body(const OpfDims& d, const DevNet& net,
                                          const double* __restrict__ x,
                                          const double* __restrict__ w,
                                          double* __restrict__ out, unsigned long long* st,
                                          int64_t blk, double* sm) {
  const int64_t nrec = (int64_t)d.L * d.T;
  const int64_t r0 = blk * kBS;
  const int64_t r = r0 + threadIdx.x;
  const int nb = (int)(nrec - r0 < kBS ? nrec - r0 : kBS);
  const bool valid = r < nrec;
  double p = 0, q = 0, G = 0, B = 0, vf = 0, vt = 0, thf = 0, tht = 0;
  int64_t rk = -1;  // record of the line's thermal pattern (12: p^2 + q^2 <= smax^2), if rated
  bool loop = false;  // a self-loop line (from == to)
  if (valid) {
    const int32_t l = (int32_t)(r / d.T), t = (int32_t)(r - (int64_t)l * d.T);
    const int32_t f = __ldg(net.lf + l), to = __ldg(net.lt + l);
    loop = f == to;
    const int32_t k = __ldg(net.l_therm + l);
    if (k >= 0) rk = (int64_t)k * d.T + t;
    G = __ldg(net.lg + l);
    B = __ldg(net.lb + l);
    p = x[d.p0 + r];
    q = x[d.q0 + r];
    vf = x[d.v0 + (int64_t)f * d.T + t];
    vt = x[d.v0 + (int64_t)to * d.T + t];
    thf = x[d.th0 + (int64_t)f * d.T + t];
    tht = x[d.th0 + (int64_t)to * d.T + t];
  }
  const LineState ls = line_state(G, B, vf, vt, thf, tht);

  if constexpr (MODE == EV_G) {
    if (valid) {
      const double gp = g_flow_p(ls, G, p);
      const double gq = g_flow_q(ls, B, q);
      const double ga = thf - tht;
      out[d.flow_p0 + r] = gp;
      out[d.flow_q0 + r] = gq;
      out[d.ang0 + r] = ga;
      if (!isfinite(gp)) report(st, d.pid[K_FLOW_P], r);
      if (!isfinite(gq)) report(st, d.pid[K_FLOW_Q], r);
      if (!isfinite(ga)) report(st, d.pid[K_ANGLE], r);
      if (rk >= 0) {  // thermal row of the same (line, period)
        const double v = g_thermal(p, q);
        out[d.therm0 + rk] = v;
        if (!isfinite(v)) report(st, d.pid[K_THERMAL], rk);
      }
    }
  } else if constexpr (MODE == EV_J) {
    // balance flows: (+1 to-record, -1 from-record); angle: (1, -1)
    const double pm[2] = {1.0, -1.0};
    const_out<2>(out + d.jac_off[K_BAL_P_FLOW] + 2 * r0, nb, pm);
    const_out<2>(out + d.jac_off[K_BAL_Q_FLOW] + 2 * r0, nb, pm);
    const_out<2>(out + d.jac_off[K_ANGLE] + 2 * r0, nb, pm);
    double jp[5], jq[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      jp[i] = j_flow_p(ls, G, B, i);
      jq[i] = j_flow_q(ls, G, B, i);
    }
    if (valid) {
      bool okp = true, okq = true;
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        okp = okp && isfinite(jp[i]);
        okq = okq && isfinite(jq[i]);
      }
      if (!okp) report(st, d.pid[K_FLOW_P], r);
      if (!okq) report(st, d.pid[K_FLOW_Q], r);
    }
    stage_out<5>(sm, jp, valid, out + d.jac_off[K_FLOW_P] + 5 * r0, nb);
    stage_out<5>(sm, jq, valid, out + d.jac_off[K_FLOW_Q] + 5 * r0, nb);
    if (rk >= 0) {  // thermal [p, q]: (2p, 2q)
      const double j0 = j_thermal(p), j1 = j_thermal(q);
      out[d.jac_off[K_THERMAL] + 2 * rk] = j0;
      out[d.jac_off[K_THERMAL] + 2 * rk + 1] = j1;
      if (!(isfinite(j0) && isfinite(j1))) report(st, d.pid[K_THERMAL], rk);
    }
  } else {  // EV_H
    const double z2[2] = {0.0, 0.0};
    const double z3[3] = {0.0, 0.0, 0.0};
    const_out<2>(out + d.hess_off[K_BAL_P_FLOW] + 2 * r0, nb, z2);
    const_out<2>(out + d.hess_off[K_BAL_Q_FLOW] + 2 * r0, nb, z2);
    const_out<3>(out + d.hess_off[K_ANGLE] + 3 * r0, nb, z3);
    double wp = 0.0, wq = 0.0;
    if (valid) {
      wp = w[d.flow_p0 + r];
      wq = w[d.flow_q0 + r];
    }
    double hp[15], hq[15];
#pragma unroll
    for (int i = 0; i < 15; ++i) {
      hp[i] = h_flow_p(ls, G, wp, i);
      hq[i] = h_flow_q(ls, B, wq, i);
    }
    if (loop) {  // v_f == v_t and th_f == th_t: the mirrored local entries (v_t, v_f) and
                 // (th_t, th_f) fold onto one diagonal slot -- double_slots, doubled as the
                 // reference does (pattern_model.hpp:193-197, 433)
      hp[6] += hp[6];
      hp[13] += hp[13];
      hq[6] += hq[6];
      hq[13] += hq[13];
    }
    if (valid) {
      bool okp = true, okq = true;
#pragma unroll
      for (int i = 0; i < 15; ++i) {
        okp = okp && isfinite(hp[i]);
        okq = okq && isfinite(hq[i]);
      }
      if (!okp) report(st, d.pid[K_FLOW_P], r);
      if (!okq) report(st, d.pid[K_FLOW_Q], r);
    }
    stage_out<15>(sm, hp, valid, out + d.hess_off[K_FLOW_P] + 15 * r0, nb);
    stage_out<15>(sm, hq, valid, out + d.hess_off[K_FLOW_Q] + 15 * r0, nb);
    if (rk >= 0) {  // thermal: (2a, 0, 2a), a = the row weight (zeros when a == 0)
      const double a = w[d.therm0 + rk];
      double h0 = 0.0;
      if (a != 0.0) {
        h0 = h_thermal_diag(a);
        if (!(isfinite(h0) && isfinite(p) && isfinite(q))) report(st, d.pid[K_THERMAL], rk);
      }
      double* o = out + d.hess_off[K_THERMAL] + 3 * rk;
      o[0] = h0;
      o[1] = 0.0;
      o[2] = h0;
    }
  }
}

// ------------------------------------------------------------- generators
// Pattern 0 (cost: f, grad, H) and 3, 4 (injections: J = 1, H = 0).
// EV_F: each block reduces its records in a fixed tree into fpart[blk]; the last
// block to finish (completion counter) sums the partials in a fixed order --
// contiguous per-thread chunks, then a tree -- and resets the counter, so f is
// independent of block scheduling.
template <int MODE>
__device__ __forceinline__ void gen_body(const OpfDims& d, const DevNet& net,
                                         const double* __restrict__ x, double ow,
                                         double* __restrict__ out, double* __restrict__ fpart,
                                         unsigned int* cnt, unsigned long long* st, int64_t blk,
                                         int64_t nblk_gen) {
  const int64_t nrec = (int64_t)d.G * d.T;
  const int64_t r0 = blk * kBS;
  const int64_t r = r0 + threadIdx.x;
  const int nb = (int)(nrec - r0 < kBS ? nrec - r0 : kBS);
  const bool valid = r < nrec;
  double pg = 0.0, c2 = 0.0, c1 = 0.0, c0 = 0.0;
  if (valid) {
    const int32_t g = (int32_t)(r / d.T);
    pg = x[d.pg0 + r];
    c2 = __ldg(net.c2 + g);
    c1 = __ldg(net.c1 + g);
    c0 = __ldg(net.c0 + g);
  }
  if constexpr (MODE == EV_F) {
    __shared__ double red[kBS];
    __shared__ bool last;
    // ((c2*pg^2) + (c1*pg)) + c0, opf.hpp:245; partial sums in a fixed tree
    double v = 0.0;
    if (valid) {
      v = f_cost(c2, c1, c0, pg);
      if (!isfinite(v)) report(st, d.pid[K_COST], r);
    }
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = kBS / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      fpart[blk] = red[0];
      __threadfence();
      last = atomicAdd(cnt, 1u) == (unsigned int)(nblk_gen - 1);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      const int n = (int)nblk_gen, chunk = (n + kBS - 1) / kBS;
      const int lo = threadIdx.x * chunk, hi = min(n, lo + chunk);
      double a = 0.0;
      for (int i = lo; i < hi; ++i) a += __ldcg(fpart + i);
      red[threadIdx.x] = a;
      __syncthreads();
      for (int s = kBS / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        *out = red[0];
        *cnt = 0u;
      }
    }
  } else if constexpr (MODE == EV_GRAD) {
    if (valid) {
      const double gr = grad_cost(c2, c1, pg);  // reverse sweep order
      out[d.pg0 + r] = gr;
      if (!isfinite(gr)) report(st, d.pid[K_COST], r);
    }
  } else if constexpr (MODE == EV_J) {
    if (valid) {
      out[d.jac_off[K_BAL_P_INJ] + r] = 1.0;
      out[d.jac_off[K_BAL_Q_INJ] + r] = 1.0;
    }
  } else if constexpr (MODE == EV_H) {
    if (valid) {
      double h = 0.0;
      if (ow != 0.0) {
        h = h_cost(ow, c2);
        if (!isfinite(h) || !isfinite(pg)) report(st, d.pid[K_COST], r);
      }
      out[d.hess_off[K_COST] + r] = h;
      out[d.hess_off[K_BAL_P_INJ] + r] = 0.0;
      out[d.hess_off[K_BAL_Q_INJ] + r] = 0.0;
    }
  }
  (void)nb;
}

// ----------------------------------------------------------------- thermal
// Pattern 9: p^2 + q^2 over rated lines (opf.hpp:323-332).

// -------------------------------------------------------------------- ramp
// Pattern 11: pg(g,t) - pg(g,t-1), t = 1..T-1 (opf.hpp:343-351).
template <int MODE>
__device__ __forceinline__ void ramp_body(const OpfDims& d, const DevNet& net,
                                          const double* __restrict__ x,
                                          double* __restrict__ out, unsigned long long* st,
                                          int64_t blk) {
  const int32_t Tm = d.R;
  const int64_t nrec = (int64_t)d.GR * (Tm > 0 ? Tm : 0);
  const int64_t r0 = blk * kBS;
  const int64_t r = r0 + threadIdx.x;
  const int nb = (int)(nrec - r0 < kBS ? nrec - r0 : kBS);
  if constexpr (MODE == EV_G) {
    if (r < nrec) {
      const int32_t k = (int32_t)(r / Tm), s = d.s_lo + (int32_t)(r - (int64_t)k * Tm);
      const int32_t g = __ldg(net.ramp_gen + k);
      const double v = x[ramp_var(d, g, k, s, true)] - x[ramp_var(d, g, k, s, false)];
      out[d.ramp0 + r] = v;
      if (!isfinite(v)) report(st, d.pid[K_RAMP], r);
    }
  } else if constexpr (MODE == EV_J) {
    const double pm[2] = {1.0, -1.0};
    const_out<2>(out + d.jac_off[K_RAMP] + 2 * r0, nb, pm);
  } else {
    const double z3[3] = {0.0, 0.0, 0.0};
    const_out<3>(out + d.hess_off[K_RAMP] + 3 * r0, nb, z3);
  }
}

// --------------------------------------------------------------------- bus
// Balance rows (n,t): 0 (+) lines by ascending l (+) generators (+) loads —
// exactly the order the reference's pattern-by-pattern `g[row] += contrib`
// produces (pattern_model.hpp:307-324), so the sums are bit-identical.
__device__ __forceinline__ void bus_body(const OpfDims& d, const DevNet& net,
                                         const double* __restrict__ x, double* __restrict__ g,
                                         unsigned long long* st, int64_t blk) {
  const int64_t r = blk * kBS + threadIdx.x;
  if (r >= (int64_t)d.N * d.T) return;
  const int32_t n = (int32_t)(r / d.T), t = (int32_t)(r - (int64_t)n * d.T);
  double ap = 0.0, aq = 0.0;
  const int32_t b0 = __ldg(net.bl_ptr + n), b1 = __ldg(net.bl_ptr + n + 1);
  for (int32_t i = b0; i < b1; ++i) {
    const int32_t e = __ldg(net.bl + i);
    const int32_t l = e >> 1, side = e & 1;
    const int64_t lt = (int64_t)l * d.T + t;
    const double p = x[d.p0 + lt], q = x[d.q0 + lt];
    const double sp = side ? -p : p, sq = side ? -q : q;  // real(0)*var(0), s = -/+1
    ap += sp;
    aq += sq;
    if (!isfinite(sp)) report(st, d.pid[K_BAL_P_FLOW], 2 * lt + side);
    if (!isfinite(sq)) report(st, d.pid[K_BAL_Q_FLOW], 2 * lt + side);
  }
  const int32_t g0 = __ldg(net.bg_ptr + n), g1 = __ldg(net.bg_ptr + n + 1);
  for (int32_t i = g0; i < g1; ++i) {
    const int64_t gt = (int64_t)__ldg(net.bg + i) * d.T + t;
    const double pg = x[d.pg0 + gt], qg = x[d.qg0 + gt];
    ap += pg;
    aq += qg;
    if (!isfinite(pg)) report(st, d.pid[K_BAL_P_INJ], gt);
    if (!isfinite(qg)) report(st, d.pid[K_BAL_Q_INJ], gt);
  }
  const int32_t l0 = __ldg(net.bd_ptr + n), l1 = __ldg(net.bd_ptr + n + 1);
  for (int32_t i = l0; i < l1; ++i) {
    const int64_t jt = (int64_t)__ldg(net.bd + i) * d.T + t;
    const double pd = -net.pd[jt], qd = -net.qd[jt];
    ap += pd;
    aq += qd;
    if (!isfinite(pd)) report(st, d.pid[K_BAL_P_LOAD], jt);
    if (!isfinite(qd)) report(st, d.pid[K_BAL_Q_LOAD], jt);
  }
  g[d.bal_p0 + r] = ap;
  g[d.bal_q0 + r] = aq;
}

// ------------------------------------------------------------------ kernel
// Block ranges of one callback launch, in grid order.
struct EvalSegs {
  int64_t line, bus, ramp, gen;
};

// MODE = EV_F / EV_GRAD / EV_G / EV_J / EV_H, or EV_FG (the line-search trial:
// the EV_G classes plus the objective, `out` = g, `fout` = f).  The class branch
// is block-uniform, so the bodies' barriers are safe.
template <int MODE>
__global__ void __launch_bounds__(kBS) k_eval(OpfDims d, DevNet net, const double* __restrict__ x,
                                              const double* __restrict__ w, double ow,
                                              double* __restrict__ out, double* __restrict__ fout,
                                              double* __restrict__ fpart, unsigned int* cnt,
                                              unsigned long long* st, EvalSegs sg) {
  constexpr int CM = MODE == EV_FG ? EV_G : MODE;  // mode of the constraint classes
  constexpr bool cons = CM == EV_G || CM == EV_J || CM == EV_H;
  int64_t b = blockIdx.x;
  // the trial launch runs its latency-bound balance-row blocks first (0.125 -> 0.123 ms at
  // 30k x 96); the g launch of the step keeps them after the line stream (bus-first there
  // costs 9241 x 48 1%)
  constexpr bool bus_first = GN_G_BUS_FIRST && MODE == EV_FG;
  if constexpr (bus_first) {
    if (b < sg.bus) {
      bus_body(d, net, x, out, st, b);
      return;
    }
    b -= sg.bus;
  }
  if constexpr (cons) {
    if (b < sg.line) {
      if constexpr (CM == EV_G) {
        line_body<EV_G>(d, net, x, w, out, st, b, nullptr);
      } else {
        __shared__ __align__(16) double sm[kBS * 15 + 2];
        line_body<CM>(d, net, x, w, out, st, b, sm);
      }
      return;
    }
    b -= sg.line;
  }
  if constexpr (CM == EV_G && !bus_first) {
    if (b < sg.bus) {
      bus_body(d, net, x, out, st, b);
      return;
    }
    b -= sg.bus;
  }
  if constexpr (cons) {
    if (b < sg.ramp) {
      ramp_body<CM>(d, net, x, out, st, b);
      return;
    }
    b -= sg.ramp;
  }
  if constexpr (MODE == EV_FG) gen_body<EV_F>(d, net, x, ow, fout, fpart, cnt, st, b, sg.gen);
  else if constexpr (MODE != EV_G) gen_body<MODE>(d, net, x, ow, out, fpart, cnt, st, b, sg.gen);
}

// All five callbacks of an IPM iteration in ONE launch (gn_eval_all): the block ranges of
// k_eval<H>, <J>, <G>, <GRAD>, <F> concatenated (heavy line streams first, the short
// generator / ramp / zero-fill blocks in the tail), one shared staging buffer for the J and
// H record blocks.  Same bodies, so every output is bit-identical to the five launches.
struct AllSegs {
  int64_t hl, jl, gl, gb, hr, jr, gr, hg, jg, dg, fg, dz;
};
struct AllOut {
  double *f, *grad, *g, *jac, *hess;
};
constexpr int kZeroPerBlock = kBS * 8;  // grad zero-fill: doubles per block
// the single launch up to this many blocks (1354 x 24: ~1.7k blocks, step -12%; 9241 x 48:
// ~17k, five launches better)
#ifndef GN_EVAL_ALL_MAXBLK
#define GN_EVAL_ALL_MAXBLK 6000
#endif
__global__ void __launch_bounds__(kBS) k_eval_all(OpfDims d, DevNet net,
                                                  const double* __restrict__ x,
                                                  const double* __restrict__ w, double ow,
                                                  AllOut o, double* __restrict__ fpart,
                                                  unsigned int* cnt, unsigned long long* st,
                                                  AllSegs sg) {
  __shared__ __align__(16) double sm[kBS * 15 + 2];
  int64_t b = blockIdx.x;
  if (b < sg.hl) return line_body<EV_H>(d, net, x, w, o.hess, st, b, sm);
  b -= sg.hl;
  if (b < sg.jl) return line_body<EV_J>(d, net, x, w, o.jac, st, b, sm);
  b -= sg.jl;
  if (b < sg.gl) return line_body<EV_G>(d, net, x, w, o.g, st, b, nullptr);
  b -= sg.gl;
  if (b < sg.gb) return bus_body(d, net, x, o.g, st, b);
  b -= sg.gb;
  if (b < sg.hr) return ramp_body<EV_H>(d, net, x, o.hess, st, b);
  b -= sg.hr;
  if (b < sg.jr) return ramp_body<EV_J>(d, net, x, o.jac, st, b);
  b -= sg.jr;
  if (b < sg.gr) return ramp_body<EV_G>(d, net, x, o.g, st, b);
  b -= sg.gr;
  if (b < sg.hg) return gen_body<EV_H>(d, net, x, ow, o.hess, fpart, cnt, st, b, sg.hg);
  b -= sg.hg;
  if (b < sg.jg) return gen_body<EV_J>(d, net, x, ow, o.jac, fpart, cnt, st, b, sg.jg);
  b -= sg.jg;
  if (b < sg.dg) return gen_body<EV_GRAD>(d, net, x, ow, o.grad, fpart, cnt, st, b, sg.dg);
  b -= sg.dg;
  if (b < sg.fg) return gen_body<EV_F>(d, net, x, ow, o.f, fpart, cnt, st, b, sg.fg);
  b -= sg.fg;
  // the gradient's non-generator blocks are zero (pattern_model.hpp:336 zero-fills)
  const int64_t z0 = d.qg0 + b * kZeroPerBlock, z1 = min((int64_t)d.n, z0 + kZeroPerBlock);
  for (int64_t i = z0 + threadIdx.x; i < z1; i += kBS) o.grad[i] = 0.0;
}

// ------------------------------------------------------------------ driver
static unsigned nblk(int64_t n) { return (unsigned)((n + kBS - 1) / kBS); }

static const char* eval_name(int mode) {
  switch (mode) {
    case EV_F: return "k_eval<F>";
    case EV_GRAD: return "k_eval<GRAD>";
    case EV_G: return "k_eval<G>";
    case EV_J: return "k_eval<J>";
    case EV_H: return "k_eval<H>";
    default: return "k_eval<FG>";
  }
}

// the completion counter of the objective's last-block sum lives after the partials
static unsigned int* fcount(const OpfDims& d, double* fpart) {
  return reinterpret_cast<unsigned int*>(fpart + nblk((int64_t)d.G * d.T));
}

void launch_eval(int mode, const OpfDims& d, const DevNet& net, const double* x,
                 const double* w, double ow, double* out, double* fpart,
                 unsigned long long* st, cudaStream_t s, double* fout) {
  const int64_t nl = (int64_t)d.L * d.T, ng = (int64_t)d.G * d.T,
                nr = d.pid[K_RAMP] >= 0 ? (int64_t)d.GR * d.R : 0,
                nb = (int64_t)d.N * d.T;
  EvalSegs sg{0, 0, 0, 0};
  const bool wants_f = mode == EV_F || mode == EV_FG;
  if (mode == EV_FG || mode == EV_G || mode == EV_J || mode == EV_H) {
    sg.line = nblk(nl);
    sg.ramp = nblk(nr);
  }
  if (mode == EV_FG || mode == EV_G) sg.bus = nblk(nb);
  if (mode != EV_G) sg.gen = nblk(ng);
  if (mode == EV_GRAD && d.n > d.qg0)  // zero the non-generator blocks; the kernel writes pg
    GN_CK(cudaMemsetAsync(out + d.qg0, 0, sizeof(double) * (d.n - d.qg0), s));
  double* fo = mode == EV_FG ? fout : out;
  if (wants_f && !sg.gen) GN_CK(cudaMemsetAsync(fo, 0, sizeof(double), s));  // no generators
  const int64_t blocks = sg.line + sg.bus + sg.ramp + sg.gen;
  if (blocks) {
    KTimer kt(eval_name(mode), s);
    unsigned int* cnt = fcount(d, fpart);
    const dim3 grid((unsigned)blocks);
    switch (mode) {
      case EV_F: k_eval<EV_F><<<grid, kBS, 0, s>>>(d, net, x, w, ow, out, fout, fpart, cnt, st, sg); break;
      case EV_GRAD: k_eval<EV_GRAD><<<grid, kBS, 0, s>>>(d, net, x, w, ow, out, fout, fpart, cnt, st, sg); break;
      case EV_G: k_eval<EV_G><<<grid, kBS, 0, s>>>(d, net, x, w, ow, out, fout, fpart, cnt, st, sg); break;
      case EV_J: k_eval<EV_J><<<grid, kBS, 0, s>>>(d, net, x, w, ow, out, fout, fpart, cnt, st, sg); break;
      case EV_H: k_eval<EV_H><<<grid, kBS, 0, s>>>(d, net, x, w, ow, out, fout, fpart, cnt, st, sg); break;
      default: k_eval<EV_FG><<<grid, kBS, 0, s>>>(d, net, x, w, ow, out, fout, fpart, cnt, st, sg); break;
    }
    count_launch();
  }
  GN_CK(cudaGetLastError());
}

void launch_eval_all(const OpfDims& d, const DevNet& net, const double* x, const double* w,
                     double ow, double* f, double* grad, double* g, double* jac, double* hess,
                     double* fpart, unsigned long long* st, cudaStream_t s) {
  const int64_t nl = (int64_t)d.L * d.T, ng = (int64_t)d.G * d.T,
                nr = d.pid[K_RAMP] >= 0 ? (int64_t)d.GR * d.R : 0,
                nb = (int64_t)d.N * d.T;
  AllSegs sg{};
  sg.hl = sg.jl = sg.gl = nblk(nl);
  sg.gb = nblk(nb);
  sg.hr = sg.jr = sg.gr = nblk(nr);
  sg.hg = sg.jg = sg.dg = sg.fg = nblk(ng);
  sg.dz = d.n > d.qg0 ? (d.n - d.qg0 + kZeroPerBlock - 1) / kZeroPerBlock : 0;
  const int64_t blocks = sg.hl + sg.jl + sg.gl + sg.gb + sg.hr + sg.jr + sg.gr + sg.hg + sg.jg +
                         sg.dg + sg.fg + sg.dz;
  if (blocks > GN_EVAL_ALL_MAXBLK) {
    // large problems: the five launches (each callback's own occupancy; the single launch
    // gives every block the J / H staging buffer: 30k x 96 +3.6%, 9241 x 48 +0.4%)
    launch_eval(EV_F, d, net, x, w, ow, f, fpart, st, s);
    launch_eval(EV_GRAD, d, net, x, w, ow, grad, fpart, st, s);
    launch_eval(EV_G, d, net, x, w, ow, g, fpart, st, s);
    launch_eval(EV_J, d, net, x, w, ow, jac, fpart, st, s);
    launch_eval(EV_H, d, net, x, w, ow, hess, fpart, st, s);
    return;
  }
  if (!sg.fg) GN_CK(cudaMemsetAsync(f, 0, sizeof(double), s));  // no generators
  if (blocks) {
    KTimer kt("k_eval<ALL>", s);
    k_eval_all<<<(unsigned)blocks, kBS, 0, s>>>(d, net, x, w, ow, AllOut{f, grad, g, jac, hess},
                                                fpart, fcount(d, fpart), st, sg);
    count_launch();
  }
  GN_CK(cudaGetLastError());
}

// objective partials + one completion counter (zeroed at context creation)
size_t fpart_size(const OpfDims& d) { return nblk((int64_t)d.G * d.T) + 2; }

}  // namespace gnb
