// Device-resident IPM vector operations (gn_ipm.cu); ABI in gn_api.cu.
#pragma once
#include "gn_kkt.cuh"

struct gn_ipm {
  int device = 0;
  gn_kkt* K = nullptr;
  int32_t n = 0, m = 0;
  int64_t nj = 0;
  gnb::DBuf<double> xl, xu, sl, su;
  gnb::Csc jt;  // per column of J: COO indices ascending (J^T y)
  gnb::Csc jr;  // per row of J: COO indices ascending (J x)
  gnb::Csc at;  // per column of A: CSR positions, rows ascending (A^T v)
  // flattened lists for the product kernels: [begin, end) of each list in src order and
  // the other index (row for columns, column for rows) of each contributor, so a thread's
  // loads are two levels deep (list bounds, then src/other, then the values)
  gnb::DBuf<int2> jt_be, jr_be, at_be;
  gnb::DBuf<int32_t> jt_oth, jr_oth, at_oth;
  gnb::DBuf<double> part;  // reduction partials
  gnb::DBuf<double> scratch;
};

namespace gnb {
gn_ipm* ipm_create(gn_kkt* K, const double* xl, const double* xu, const double* sl,
                   const double* su, bool device_in);
void ipm_jac_t(gn_ipm* P, const double* jv, const double* y, double* out, cudaStream_t s);
void ipm_jac(gn_ipm* P, const double* jv, const double* x, double* out, cudaStream_t s);
void ipm_residuals(gn_ipm* P, const gn_iterate& it, const double* grad, const double* g,
                   const double* jv, double mu, const gn_residuals& r, cudaStream_t s);
void ipm_condense(gn_ipm* P, const gn_iterate& it, const gn_residuals& r, double* sx, double* ss,
                  double* qx, double* qs, cudaStream_t s);
void ipm_recover(gn_ipm* P, const gn_iterate& it, const gn_residuals& r, const gn_direction& d,
                 cudaStream_t s);
void ipm_kkt_error(gn_ipm* P, const gn_iterate& it, const gn_residuals& r, double mu, double* out,
                   cudaStream_t s);
void ipm_barrier(gn_ipm* P, double f, const double* x, const double* sv, double mu, double* out,
                 cudaStream_t s);
void ipm_slope(gn_ipm* P, const double* grad, const gn_iterate& it, const gn_direction& d,
               double mu, double* out, cudaStream_t s);
void ipm_violation(gn_ipm* P, const double* g, const double* sv, double* out, cudaStream_t s);
void ipm_ftb(gn_ipm* P, const gn_iterate& it, const gn_direction& d, double tau, double* out,
             cudaStream_t s);
void kkt_solve_rhs(gn_ipm* P, const double* qx, const double* qs, const double* qy,
                   const double* ss, double dw, double dc, double* rhs, double* tm,
                   cudaStream_t s);
void kkt_solve_finish(gn_ipm* P, const double* dx, const double* qs, const double* qy,
                      const double* ss, double dw, double dc, double* ds, double* dy,
                      cudaStream_t s);
}  // namespace gnb
