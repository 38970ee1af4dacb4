#pragma once
#include "gn_internal.cuh"

namespace gnb {

// EV_FG: the line-search trial, g into `out` and f into `fout`, one launch
enum EvalMode { EV_F = 0, EV_GRAD = 1, EV_G = 2, EV_J = 3, EV_H = 4, EV_FG = 5 };

// Enqueue one callback (one kernel, plus a memset for EV_GRAD) on stream s;
// failures are latched into *st.  fpart: fpart_size(d) doubles, zeroed once.
void launch_eval(int mode, const OpfDims& d, const DevNet& net, const double* x,
                 const double* w, double ow, double* out, double* fpart,
                 unsigned long long* st, cudaStream_t s, double* fout = nullptr);
size_t fpart_size(const OpfDims& d);
// f, grad, g, J and H(w, ow) in one launch (gn_eval_all), bit-identical to five launch_eval
void launch_eval_all(const OpfDims& d, const DevNet& net, const double* x, const double* w,
                     double ow, double* f, double* grad, double* g, double* jac, double* hess,
                     double* fpart, unsigned long long* st, cudaStream_t s);

void build_structure(gn_ctx* c, int32_t* jr, int32_t* jc, int32_t* hr, int32_t* hc);
void build_lifted(gn_ctx* c);
void host_bounds(const gn_ctx* c, double* xl, double* xu, double* xs, double* rl,
                 double* ru);
int32_t exclusive_scan(const int32_t* flag, int32_t* pos, int64_t n, cudaStream_t s);
int64_t launch_count();
void profile_enable(bool on);
bool profiling();
void profile_reset();
int profile_count();
const char* profile_get(int i, double* ms, int64_t* launches);

}  // namespace gnb
