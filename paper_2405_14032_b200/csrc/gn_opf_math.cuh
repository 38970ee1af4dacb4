// Closed-form values of the OPF patterns, shared by the
// callback kernels (gn_eval.cu) and the fused KKT kernels (gn_opf_fused.cu):
// one source expression per value, compiled with -fmad=false, so a value
// recomputed inside a fused kernel is bit-identical to the one the callback
// wrote.  Value/Jacobian expressions follow the reference tape's operation
// order (opf.hpp:310-319 forward; tape.hpp:168-210 reverse sweep).
#pragma once
#include <cuda_runtime.h>

namespace gnb {

// Per (line, period) trigonometric state.  dth = th_f - th_t.
struct LineState {
  double vf, vt, vfvt, cs, sn, Cs, Sn;
};

__device__ __forceinline__ LineState line_state(double G, double B, double vf, double vt,
                                                double thf, double tht) {
  LineState s;
  s.vf = vf;
  s.vt = vt;
  s.vfvt = vf * vt;
  sincos(thf - tht, &s.sn, &s.cs);
  s.Cs = G * s.cs + B * s.sn;  // flow_p tape node 17: G cos + B sin
  s.Sn = G * s.sn - B * s.cs;  // flow_q tape node 18: G sin - B cos
  return s;
}

// ---- g (forward sweep order)
__device__ __forceinline__ double g_flow_p(const LineState& s, double G, double p) {
  return p - (G * (s.vf * s.vf) - s.vfvt * s.Cs);
}
__device__ __forceinline__ double g_flow_q(const LineState& s, double B, double q) {
  return q - ((-B) * (s.vf * s.vf) - s.vfvt * s.Sn);
}

// ---- J (reverse sweep order), fields [flow, v_f, v_t, th_f, th_t]
__device__ __forceinline__ double j_flow_p(const LineState& s, double G, double B, int f) {
  switch (f) {
    case 0: return 1.0;
    case 1: return s.Cs * s.vt + ((-G) * 2.0) * s.vf;
    case 2: return s.Cs * s.vf;
    case 3: return (s.vfvt * B) * s.cs - (s.vfvt * G) * s.sn;
    default: return -((s.vfvt * B) * s.cs - (s.vfvt * G) * s.sn);
  }
}
__device__ __forceinline__ double j_flow_q(const LineState& s, double G, double B, int f) {
  switch (f) {
    case 0: return 1.0;
    case 1: return s.Sn * s.vt + (B * 2.0) * s.vf;
    case 2: return s.Sn * s.vf;
    case 3: return (s.vfvt * B) * s.sn + (s.vfvt * G) * s.cs;
    default: return -((s.vfvt * B) * s.sn + (s.vfvt * G) * s.cs);
  }
}

// ---- H (lower triangle, local slot order (0,0)(1,0)..(4,0)(1,1)..(4,1)(2,2)..(4,4)),
// already multiplied by the row weight a; a == 0 -> 0 (pattern_model.hpp:409-412).
// Slots 0-4 and 9 are identically zero.
__device__ __forceinline__ double h_flow_p(const LineState& s, double G, double a, int slot) {
  if (a == 0.0) return 0.0;
  switch (slot) {
    case 5: return ((-2.0) * G) * a;          // (v_f, v_f)
    case 6: return s.Cs * a;                  // (v_t, v_f)
    case 7: return -((s.vt * s.Sn) * a);      // (th_f, v_f)
    case 8: return (s.vt * s.Sn) * a;         // (th_t, v_f)
    case 10: return -((s.vf * s.Sn) * a);     // (th_f, v_t)
    case 11: return (s.vf * s.Sn) * a;        // (th_t, v_t)
    case 12: return -((s.vfvt * s.Cs) * a);   // (th_f, th_f)
    case 13: return (s.vfvt * s.Cs) * a;      // (th_t, th_f)
    case 14: return -((s.vfvt * s.Cs) * a);   // (th_t, th_t)
    default: return 0.0;
  }
}
__device__ __forceinline__ double h_flow_q(const LineState& s, double B, double a, int slot) {
  if (a == 0.0) return 0.0;
  switch (slot) {
    case 5: return (2.0 * B) * a;
    case 6: return s.Sn * a;
    case 7: return (s.vt * s.Cs) * a;
    case 8: return -((s.vt * s.Cs) * a);
    case 10: return (s.vf * s.Cs) * a;
    case 11: return -((s.vf * s.Cs) * a);
    case 12: return -((s.vfvt * s.Sn) * a);
    case 13: return (s.vfvt * s.Sn) * a;
    case 14: return -((s.vfvt * s.Sn) * a);
    default: return 0.0;
  }
}

// thermal p^2 + q^2: J = (2p, 2q), H = (2a, 0, 2a)
__device__ __forceinline__ double g_thermal(double p, double q) { return p * p + q * q; }
__device__ __forceinline__ double j_thermal(double v) { return 2.0 * v; }
__device__ __forceinline__ double h_thermal_diag(double a) { return a == 0.0 ? 0.0 : (a * 2.0); }

// cost ((c2 pg^2) + c1 pg) + c0: grad c1 + (2 c2) pg, H (ow c2) 2
__device__ __forceinline__ double f_cost(double c2, double c1, double c0, double pg) {
  return (c2 * (pg * pg) + c1 * pg) + c0;
}
__device__ __forceinline__ double grad_cost(double c2, double c1, double pg) {
  return c1 + (c2 * 2.0) * pg;
}
__device__ __forceinline__ double h_cost(double ow, double c2) {
  return ow == 0.0 ? 0.0 : (ow * c2) * 2.0;
}

// condensed.hpp:112-116: d = sd / (1 + dc sd) computed as sd * (1 / (1 + dc sd))
__device__ __forceinline__ double dvec(double sigma_s, double dw, double dc) {
  const double sd = sigma_s + dw;
  const double c = 1.0 / (1.0 + dc * sd);
  return sd * c;
}
// one AtDA pair term: (d * A[ka]) * A[kb]  (condensed.hpp:126-129)
__device__ __forceinline__ double pair_term(double d, double aka, double akb) {
  const double va = d * aka;
  return va * akb;
}

}  // namespace gnb
