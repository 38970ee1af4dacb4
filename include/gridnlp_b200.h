/* include/gridnlp_b200.h — the drop-in C-ABI of the B200 hot path.
 *
 * Pure C: opaque handles, plain pointers and sizes, int32 indices (the
 * reference's index_t, common.hpp:14).  Every entry point returns an int
 * status (GN_OK = 0) and, where it can fail, fills a caller-provided gn_error.
 *
 * Each function names the reference interface it replaces (paths relative to
 * /root/reference/proj/include/gridnlp).  The C++ adapters that put this ABI
 * back behind the reference's own classes are
 *   include/gridnlp_b200/cuda_opf_nlp.hpp   -> ipm::NlpProblem   (ipm/nlp.hpp:15-39)
 *   include/gridnlp_b200/shim/gridnlp/ipm/condensed.hpp
 *                                           -> ipm::CondensedKkt (ipm/condensed.hpp:27-185)
 *   include/gridnlp_b200/shim/gridnlp/ipm/lifted.hpp
 *                                           -> ipm::LiftedProblem (ipm/lifted.hpp:22-200)
 * and INTEGRATION.md shows the bindings a maintainer adds.
 *
 * Memory modes (`mem` argument):
 *   GN_MEM_HOST          pointers are host memory; the call copies H2D/D2H and
 *                        returns after the result is on the host (the
 *                        reference's std::span semantics).
 *   GN_MEM_DEVICE        pointers are device memory on the context's device;
 *                        the call synchronises the context stream and returns
 *                        the evaluation status.
 *   GN_MEM_DEVICE_ASYNC  device pointers, no synchronisation: kernels are only
 *                        enqueued on the context stream; evaluation failures are
 *                        latched on the device and reported by gn_ctx_status().
 * OR-ing GN_IN_FULL into `mem` for a KKT created by gn_kkt_create_lifted() says
 * the J/H inputs are the FULL (un-lifted) callback outputs; the lifted gather
 * (lifted.hpp:249-264) is then fused into the KKT kernels.
 */
#ifndef GRIDNLP_B200_H
#define GRIDNLP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GN_ABI_VERSION 1

enum {
  GN_OK = 0,
  GN_ERR_INVALID = 1,     /* bad shape/argument: the reference throws gridnlp::Error */
  GN_ERR_EVAL = 2,        /* domain / non-finite result: the reference returns false */
  GN_ERR_CUDA = 3,        /* CUDA runtime failure (no GPU, OOM, ...) */
  GN_ERR_UNSUPPORTED = 4  /* e.g. the fused assembly on a network it cannot enumerate */
};

enum { GN_MEM_HOST = 0, GN_MEM_DEVICE = 1, GN_MEM_DEVICE_ASYNC = 2, GN_IN_FULL = 16 };

/* Failure report.  For GN_ERR_EVAL, (pattern, record) is the lexicographically
 * smallest failing (pattern id, record index) in registration order — the
 * record the reference's EvalStatus names (pattern_model.hpp:16-25, 544-571). */
typedef struct {
  int32_t code;
  int32_t pattern;
  int32_t record;
  char message[244];
} gn_error;

/* Per-unit network, the reference's NetworkData in SoA form (power/network.hpp:18-66).
 * Element cross-references are 0-based indices.  line_smax / gen_ramp use +inf
 * for "no rating" / "no ramp limit" exactly like the reference. */
typedef struct {
  int32_t n_bus, n_line, n_gen, n_load, reference_bus;
  const double *bus_vmin, *bus_vmax, *vm_start, *va_start;               /* [n_bus]  */
  const int32_t *line_from, *line_to;                                   /* [n_line] */
  const double *line_g, *line_b, *line_smax, *line_amin, *line_amax;    /* [n_line] */
  const int32_t *gen_bus;                                               /* [n_gen]  */
  const double *gen_pmin, *gen_pmax, *gen_qmin, *gen_qmax, *gen_ramp;   /* [n_gen]  */
  const double *gen_c2, *gen_c1, *gen_c0, *gen_pstart, *gen_qstart;     /* [n_gen]  */
  const int32_t *load_bus;                                              /* [n_load] */
  const double *load_p, *load_q;                                        /* [n_load] */
} gn_network;

/* Model sizes.  Full space = the NlpProblem the reference's PatternNlp exposes;
 * lifted = after LiftedProblem's fixed-variable filter (lifted.hpp:25-100). */
typedef struct {
  int64_t n_vars, n_cons, jac_nnz, hess_nnz;       /* nlp.hpp:19-30 */
  int64_t n_thermal, n_ramp_gens, periods;         /* OpfLayout (opf.hpp:29-30) */
  int64_t n_free, jac_nnz_lifted, hess_nnz_lifted; /* valid after gn_lifted_create */
} gn_sizes;

typedef struct gn_ctx gn_ctx;
typedef struct gn_kkt gn_kkt;

int gn_abi_version(void);
/* Number of CUDA kernels this library has launched (process-wide counter). */
int64_t gn_launch_count(void);
/* Per-kernel CUDA-event timing of this library's launches (bench.py roofline):
 * enable, run, then gn_profile_count() synchronises and returns the number of
 * kernels; gn_profile_get(i) returns its name, total ms and launch count. */
void gn_profile_enable(int on);
void gn_profile_reset(void);
int gn_profile_count(void);
const char* gn_profile_get(int i, double* total_ms, int64_t* launches);
/* Reports whether a usable CUDA device is present (count into *n_devices). */
int gn_device_count(int32_t* n_devices);

/* ----------------------------------------------------------------- inputs */
/* Demand multipliers, bit-identical to generate_load_profile
 * (power/network.hpp:104-140; mt19937_64, top-53-bit mapping).  scale is
 * periods x n_load, period-major (LoadProfile::scale).  Host-side utility. */
int gn_load_profile(int32_t n_load, int32_t periods, double resolution_minutes,
                    uint64_t seed, double amplitude, double noise, double* scale,
                    gn_error* err);

/* ---------------------------------------------------------------- context */
/* Builds the multi-period OPF on the device: replaces
 * power::build_multiperiod_opf (opf.hpp:100-355) + PatternModel::freeze
 * (pattern_model.hpp:158-207) + ipm::PatternNlp (pattern_nlp.hpp:15-62).
 * `scale` is the host T x n_load demand table (MultiPeriodCase::pd/qd,
 * network.hpp:166-171).  Lines with from == to are rejected (GN_ERR_UNSUPPORTED). */
int gn_ctx_create(const gn_network* net, int32_t periods, const double* scale,
                  int32_t device, gn_ctx** out, gn_error* err);
/* One period shard of a periods_total-period horizon: the
 * periods [first_period, first_period + periods), scale = that slice of the
 * demand table.  Layout = the reference layout over the shard's periods, plus
 * ghost generator set-points after the regular blocks: pg(first_period - 1)
 * (fixed; the caller writes the previous rank's values into x) and
 * pg(first_period + periods) (free; the rows using it are owned by the next
 * rank, whose sigma_s values the caller writes into the ghost rows).  The
 * ramp row of step t belongs to the rank owning period t.  With the halo
 * filled, every owned row, record and lifted M column equals the global
 * problem's, bit for bit (tests/test_shard.py). */
int gn_ctx_create_shard(const gn_network* net, int32_t periods_total, int32_t first_period,
                        int32_t periods, const double* scale, int32_t device, gn_ctx** out,
                        gn_error* err);
/* info = [t0, T_total, prev, next, n_ramp_gens, n_base, ghost_prev0, ghost_next0,
 *         ramp_row0, ramp_rows_per_gen, first_step, owned_lifted_columns (-1 before
 *         gn_lifted_create)]; ramp_gens[n_ramp_gens] (may be NULL). */
int gn_ctx_shard_info(gn_ctx* ctx, int64_t* info, int32_t* ramp_gens);

/* ---------------------------------------------------------- period-shard halo
 * The ramp coupling between period shards (opf.hpp:343-351) over peer
 * memory: each rank owns a small device region that its neighbours store into directly
 * (NVLink / NVSwitch P2P), released by a step flag -- pg(., t0-1) from rank-1, pg(., t1)
 * and the sigma_s of the step-t1 ramp rows from rank+1, and every rank's objective
 * partial.  An exchange is one kernel on the caller's stream (no host call: capturable in
 * a CUDA graph).  Ranks on different GPUs; see gn_halo_exchange_emulated for one GPU. */
typedef struct gn_halo gn_halo;
#define GN_HALO_HANDLE_BYTES 64
#define GN_HALO_SEND 1
#define GN_HALO_RECV 2
#define GN_HALO_BOTH 3
/* ctx must be the shard of `rank` of a `world`-rank partition (gn_ctx_create_shard). */
int gn_halo_create(gn_ctx* ctx, int32_t rank, int32_t world, gn_halo** out, gn_error* err);
/* This rank's region as an IPC handle (GN_HALO_HANDLE_BYTES bytes). */
int gn_halo_ipc_handle(gn_halo* halo, void* handle);
/* Map every other rank's region from the all-gathered handles (world x
 * GN_HALO_HANDLE_BYTES; this rank's own entry is ignored). */
int gn_halo_open(gn_halo* halo, const void* handles);
/* Same-process alternative: the ranks' halos (index = rank) see each other's regions
 * directly (one GPU, or GPUs with peer access enabled). */
int gn_halo_link(gn_halo* const* halos, int32_t world);
/* phase GN_HALO_SEND: pack pg(., first / last period) and sigma_s of the step-t0 rows into
 * the neighbours' regions and release the step flag; GN_HALO_RECV: wait for this step's
 * flags, write the ghost set-points into x and the ghost rows into sigma_s; BOTH: one
 * kernel.  x / sigma_s are the shard's device vectors. */
int gn_halo_exchange(gn_halo* halo, double* x, double* sigma_s, int phase, void* stream);
/* Global objective = the ranks' partials f_local[0] added in rank order (the same value on
 * every rank, run to run); device pointers, phases as above. */
int gn_halo_objective(gn_halo* halo, const double* f_local, double* f_global, int phase,
                      void* stream);
/* One GPU: every rank's exchange (GN_HALO_BOTH) in ONE cooperative launch, CTA r = rank r
 * (world <= 8, linked halos) -- the cross-rank waits are between co-resident CTAs. */
int gn_halo_exchange_emulated(gn_halo* const* halos, int32_t world, double* const* xs,
                              double* const* sigma_s, void* stream);
int gn_halo_destroy(gn_halo* halo);
int gn_ctx_destroy(gn_ctx* ctx);
/* Publish (on = 1) or withdraw (on = 0) the context's lifted structure for gn_kkt_create:
 * a KKT created from COO arrays equal to a published context's lifted J / H structure
 * (the arrays the reference's IpmSolver passes to CondensedKkt, solver.hpp:139-141) is
 * built on that context and uses the OPF-specialised kernels -- bit-identical values,
 * recognised by gn_kkt_dims dims[7] = 1.  Publishing lifts the problem when
 * gn_lifted_create has not run (slack relaxation 0: only the structure is used).
 * gn_ctx_destroy withdraws it. */
int gn_ctx_publish(gn_ctx* ctx, int on);
/* Use a caller-owned cudaStream_t (as void*) for every launch of this context; NULL
 * returns to the context's own (non-blocking) stream, which lives until gn_ctx_destroy
 * (a KKT created on it keeps using it).  NULL is "reset", never the legacy default
 * stream: to launch on the legacy default stream pass cudaStreamLegacy ((void*)0x1),
 * or cudaStreamPerThread.  Work already enqueued is synchronised first. */
int gn_ctx_set_stream(gn_ctx* ctx, void* cuda_stream);
int gn_ctx_get_stream(gn_ctx* ctx, void** cuda_stream);
/* Synchronises the stream, returns (and clears) the latched evaluation status. */
int gn_ctx_status(gn_ctx* ctx, gn_error* err);
int gn_ctx_sizes(gn_ctx* ctx, gn_sizes* out);

/* NlpProblem::x_lower/x_upper/x_start/row_lower/row_upper (nlp.hpp:21-25).
 * Host arrays of n_vars / n_cons; any pointer may be NULL. */
int gn_ctx_bounds(gn_ctx* ctx, double* x_lower, double* x_upper, double* x_start,
                  double* row_lower, double* row_upper);
/* NlpProblem::jac_rows/jac_cols (nlp.hpp:27-28), freeze order. */
int gn_jac_structure(gn_ctx* ctx, int32_t* rows, int32_t* cols, int mem);
/* NlpProblem::hess_rows/hess_cols (nlp.hpp:29-30), (max,min) lower triangle. */
int gn_hess_structure(gn_ctx* ctx, int32_t* rows, int32_t* cols, int mem);

/* ------------------------------------------------------------- callbacks */
/* NlpProblem::eval_f (nlp.hpp:32) / PatternModel::evaluate_objective
 * (pattern_model.hpp:278-300).  In device modes `out` is a device double. */
int gn_eval_f(gn_ctx* ctx, const double* x, double* out, int mem, gn_error* err);
/* NlpProblem::eval_grad (nlp.hpp:33) / evaluate_gradient (:328-359). */
int gn_eval_grad(gn_ctx* ctx, const double* x, double* out, int mem, gn_error* err);
/* NlpProblem::eval_g (nlp.hpp:34) / evaluate_constraints (:302-326). */
int gn_eval_g(gn_ctx* ctx, const double* x, double* out, int mem, gn_error* err);
/* NlpProblem::eval_jac (nlp.hpp:35) / evaluate_jacobian (:361-388). */
int gn_eval_jac(gn_ctx* ctx, const double* x, double* out, int mem, gn_error* err);
/* NlpProblem::eval_hess (nlp.hpp:36-38) / evaluate_hessian (:393-436). */
int gn_eval_hess(gn_ctx* ctx, const double* x, const double* row_weights,
                 double obj_weight, double* out, int mem, gn_error* err);

/* Line-search trial point (solver.hpp:267-304 evaluates f and g at each trial):
 * eval_f and eval_g in one call, no derivative work, one status (the
 * lexicographically first failing (pattern, record) over both). */
int gn_eval_fg(gn_ctx* ctx, const double* x, double* f, double* g, int mem, gn_error* err);
/* One IPM iteration's callbacks (solver.hpp:157-158 and 202: eval_f, eval_grad, eval_g,
 * eval_jac and eval_hess(w, ow) at the same x) in ONE kernel launch: outputs bit-identical
 * to the five calls above, the lexicographically first failure over all five reported. */
int gn_eval_all(gn_ctx* ctx, const double* x, const double* row_weights, double obj_weight,
                double* f, double* grad, double* g, double* jac, double* hess, int mem,
                gn_error* err);

/* ---------------------------------------------------------------- lifted */
/* LiftedProblem constructor filter (lifted.hpp:25-100): free map, slack
 * boxes (relative relaxation), J/H picks.  Built on the device. */
int gn_lifted_create(gn_ctx* ctx, double relax, gn_error* err);
/* Any pointer may be NULL.  free_to_full[n_free]; jr/jc/jac_pick[jac_nnz_lifted];
 * hr/hc/hess_pick[hess_nnz_lifted]; s_lower/s_upper[n_cons] (always host). */
int gn_lifted_structure(gn_ctx* ctx, int32_t* free_to_full, int32_t* jac_rows,
                        int32_t* jac_cols, int32_t* jac_pick, int32_t* hess_rows,
                        int32_t* hess_cols, int32_t* hess_pick, double* s_lower,
                        double* s_upper, int mem);
/* LiftedProblem::eval_jac / eval_hess value gathers (lifted.hpp:249-264),
 * full -> lifted, device or host. */
int gn_lifted_gather_jac(gn_ctx* ctx, const double* jac_full, double* jac_lifted, int mem);
int gn_lifted_gather_hess(gn_ctx* ctx, const double* hess_full, double* hess_lifted,
                          int mem);
/* LiftedProblem::eval_f / eval_grad / eval_g / eval_jac / eval_hess (lifted.hpp:128-159)
 * in one call each: x is the FREE-variable vector [n_free]; it is staged into the full
 * space on the device (fixed entries at their pinned values, lifted.hpp:35-45, 165-168),
 * the callback runs, and grad [n_free], J [jac_nnz_lifted] and H [hess_nnz_lifted] come
 * back already gathered (f and g [n_cons] are not lifted).  Errors as gn_eval_*.  The
 * shim LiftedProblem (include/gridnlp_b200/shim/gridnlp/ipm/lifted.hpp) calls these for a
 * CudaOpfNlp.  A period shard returns GN_ERR_UNSUPPORTED (its ghost set-points hold halo
 * values: use the full-space calls). */
int gn_lifted_eval_f(gn_ctx* ctx, const double* x_free, double* out, int mem, gn_error* err);
int gn_lifted_eval_grad(gn_ctx* ctx, const double* x_free, double* out, int mem, gn_error* err);
int gn_lifted_eval_g(gn_ctx* ctx, const double* x_free, double* out, int mem, gn_error* err);
int gn_lifted_eval_jac(gn_ctx* ctx, const double* x_free, double* out, int mem, gn_error* err);
int gn_lifted_eval_hess(gn_ctx* ctx, const double* x_free, const double* row_weights,
                        double obj_weight, double* out, int mem, gn_error* err);
int gn_lifted_eval_fg(gn_ctx* ctx, const double* x_free, double* f, double* g, int mem,
                      gn_error* err);

/* ------------------------------------------------------------ condensed KKT */
/* CondensedKkt constructor structure (condensed.hpp:29-90) on an arbitrary
 * lifted COO (host arrays): CSR(A) + jac_slots, M = Hess U AtA U diag in CSC
 * lower + hess/pair/diag slots — sorted on the device.  The LDL^T symbolic
 * phase (ldlt.hpp:34-50) is not part of this object.  When the arrays equal the lifted
 * structure of a context published with gn_ctx_publish, the KKT is built on that context
 * (OPF-specialised kernels for lifted and GN_IN_FULL inputs; dims[7] = 1). */
int gn_kkt_create(int32_t n, int32_t m, int64_t jac_nnz, const int32_t* jac_rows,
                  const int32_t* jac_cols, int64_t hess_nnz, const int32_t* hess_rows,
                  const int32_t* hess_cols, int32_t device, gn_kkt** out, gn_error* err);
/* Same structure on the context's lifted problem (after gn_lifted_create);
 * enables GN_IN_FULL inputs and the OPF-specialised assembly kernels.  The
 * KKT shares the context's stream. */
int gn_kkt_create_lifted(gn_ctx* ctx, gn_kkt** out, gn_error* err);
int gn_kkt_destroy(gn_kkt* kkt);
/* As gn_ctx_set_stream, for the KKT's launches.  NULL returns to the KKT's own stream;
 * a KKT from gn_kkt_create_lifted has none and returns to its context's own stream. */
int gn_kkt_set_stream(gn_kkt* kkt, void* cuda_stream);
/* dims = [dim, a_nnz, m_nnz, pair_count, jac_nnz, hess_nnz, n_rows, opf_ready,
 *         fused_ready] (opf_ready / fused_ready = 1 when the OPF-specialised /
 * fused kernels verified against the generic structure at creation). */
int gn_kkt_dims(gn_kkt* kkt, int64_t* dims);
/* jacobian_csr() / pattern() (condensed.hpp:93-95). Any pointer may be NULL. */
int gn_kkt_structure(gn_kkt* kkt, int32_t* rowptr, int32_t* colidx, int32_t* colptr,
                     int32_t* rowidx, int mem);
/* The private slot maps jac_slots_/hess_slots_/pair_slots_/diag_slots_ (condensed.hpp:177-180). */
int gn_kkt_slots(gn_kkt* kkt, int32_t* jac_slots, int32_t* hess_slots, int32_t* pair_slots,
                 int32_t* diag_slots, int mem);
/* CondensedKkt::set_jacobian (condensed.hpp:99-101): A = scatter(J). */
int gn_kkt_set_jacobian(gn_kkt* kkt, const double* jac_vals, int mem);
/* CondensedKkt::assemble (condensed.hpp:105-135): M = W + dw I + Sx + At D A,
 * summed per slot in the reference's order (bit-exact given equal inputs). */
int gn_kkt_assemble(gn_kkt* kkt, const double* hess_vals, const double* sigma_x,
                    const double* sigma_s, double delta_w, double delta_c, int mem);
/* Fused B200 path for lifted OPF KKTs (fused_ready): the same A and M as
 *   set_jacobian(eval_jac(x))  and  assemble(eval_hess(x, w, ow), Sx, Ss, dw, dc)
 * bit for bit, computed straight from x (and w, ow) without reading J or H.
 * x is the FULL primal vector, row_weights/sigma_s have n_cons entries,
 * sigma_x has n_free entries.  GN_ERR_UNSUPPORTED when the fused path is off. */
int gn_kkt_set_jacobian_x(gn_kkt* kkt, const double* x, int mem);
int gn_kkt_assemble_x(gn_kkt* kkt, const double* x, const double* row_weights,
                      double obj_weight, const double* sigma_x, const double* sigma_s,
                      double delta_w, double delta_c, int mem);
/* gn_kkt_set_jacobian_x + gn_kkt_assemble_x at the same x in one call (the IPM's
 * per-iteration pair, solver.hpp:213-228): identical A and M, with the flow rows of A
 * written by the flow-column kernel from the line state it already computes.  Inertia
 * retries call gn_kkt_assemble_x alone. */
int gn_kkt_update_x(gn_kkt* kkt, const double* x, const double* row_weights, double obj_weight,
                    const double* sigma_x, const double* sigma_s, double delta_w,
                    double delta_c, int mem);
/* jacobian_values() / values() (condensed.hpp:94-96).  In the device modes the
 * destinations may be any UVA-addressable memory: device buffers or pinned host
 * buffers (an asynchronous read-back overlapping later work on the stream). */
int gn_kkt_values(gn_kkt* kkt, double* a_vals, double* m_vals, int mem);
/* The device addresses of the KKT's own A and M value arrays (CSR / CSC-lower order, valid
 * until gn_kkt_destroy), for device-resident consumers that read them in place -- a device
 * factorization, or a copy engine on another stream that returns A to the host while M is
 * still being assembled.  Their contents change with the next set_jacobian / assemble call
 * on the KKT's stream: order such reads after it with an event. */
int gn_kkt_values_ptr(gn_kkt* kkt, const double** a_vals, const double** m_vals);
/* Asynchronous read-back for host solvers: start copying A and/or M (NULL skips one) into
 * page-locked host memory (gn_host_alloc / cudaHostAlloc; pageable memory makes the copy
 * synchronous) on a side stream, after the KKT's work so far, and return at once -- the copy
 * overlaps whatever the caller does next, e.g. the next assemble's uploads (PCIe is full
 * duplex).  gn_kkt_values_wait blocks until it has landed; the KKT's next set_jacobian /
 * assemble waits for it on the device.  Not for CUDA-graph capture (the side stream is
 * joined only by that next write). */
int gn_kkt_values_start(gn_kkt* kkt, double* a_vals, double* m_vals);
int gn_kkt_values_wait(gn_kkt* kkt);
/* Selects the assembly algorithm: 0 = auto, 1 = generic contributor lists,
 * 2 = OPF-specialised (lifted KKTs only). */
/* Cap the fused/specialised KKT kernels at `ctas_per_sm` resident CTAs per SM (grid-stride;
 * 0 = uncapped, the default unless GRIDNLP_B200_GRID_CAP is set).  A cap leaves SM room for
 * kernels of other streams -- e.g. the callbacks evaluated concurrently with the KKT. */
int gn_kkt_set_grid_cap(gn_kkt* kkt, int ctas_per_sm);
int gn_kkt_set_algorithm(gn_kkt* kkt, int algo);

/* compress_to_csc (sparse/matrix.hpp:45-81) of a host COO, on the device;
 * returns the compressed nnz in *nnz_out.  colptr[ncols+1], rowidx/slot_map[nnz]. */
int gn_compress_to_csc(int32_t nrows, int32_t ncols, int64_t nnz, const int32_t* rows,
                       const int32_t* cols, int32_t* colptr, int32_t* rowidx,
                       int32_t* slot_map, int32_t* nnz_out, gn_error* err);

/* ------------------------------------------ device-resident IPM vector ops
 * (SURVEY §8(f)1-2): the per-iteration vector work of ipm::IpmSolver on the
 * lifted problem of a gn_kkt_create_lifted() KKT, so that x, s, y, z and the
 * residuals stay in HBM.  Every vector argument is a device pointer (mem =
 * GN_MEM_DEVICE or GN_MEM_DEVICE_ASYNC; GN_MEM_HOST is GN_ERR_UNSUPPORTED);
 * scalar results are written to device doubles.  Sizes: n = n_free (lifted
 * variables), m = n_cons.  Element-wise results and the sparse products are
 * bit-identical to the reference (same operation order, -fmad=false); whole-
 * vector sums use a fixed reduction tree (deterministic, equal to the
 * reference's sequential sums to rounding). */
typedef struct gn_ipm gn_ipm;
typedef struct { const double *x, *s, *y, *zlx, *zux, *zls, *zus; } gn_iterate;  /* Iterate (iterate.hpp:16-19) */
typedef struct { double *px, *ps, *py, *pzlx, *pzux, *pzls, *pzus; } gn_residuals; /* Residuals (:31-34) */
typedef struct { double *dx, *ds, *dy, *dzlx, *dzux, *dzls, *dzus; } gn_direction; /* Direction (:23-26) */

/* Bounds of the lifted problem: x_lower/x_upper[n], s_lower/s_upper[m] (+-inf = absent). */
int gn_ipm_create(gn_kkt* kkt, const double* x_lower, const double* x_upper,
                  const double* s_lower, const double* s_upper, int mem, gn_ipm** out,
                  gn_error* err);
int gn_ipm_destroy(gn_ipm* ipm);
/* jac_transpose_multiply / jac_multiply (iterate.hpp:42-62) on the lifted J COO values. */
int gn_ipm_jac_transpose_multiply(gn_ipm* ipm, const double* jac_vals, const double* y,
                                  double* out_n, int mem);
int gn_ipm_jac_multiply(gn_ipm* ipm, const double* jac_vals, const double* x, double* out_m,
                        int mem);
/* compute_residuals (iterate.hpp:64-97). */
int gn_ipm_residuals(gn_ipm* ipm, const gn_iterate* it, const double* grad, const double* g,
                     const double* jac_vals, double mu, const gn_residuals* r, int mem);
/* bound_condensation (iterate.hpp:99-145): sigma_x[n], sigma_s[m], qx[n], qs[m]. */
int gn_ipm_bound_condensation(gn_ipm* ipm, const gn_iterate* it, const gn_residuals* r,
                              double* sigma_x, double* sigma_s, double* qx, double* qs, int mem);
/* fraction_to_boundary (iterate.hpp:147-198): out2 = {primal, dual}. */
int gn_ipm_fraction_to_boundary(gn_ipm* ipm, const gn_iterate* it, const gn_direction* d,
                                double tau, double* out2, int mem);
/* barrier_value (iterate.hpp:200-218); f is a host double, out a device double. */
int gn_ipm_barrier_value(gn_ipm* ipm, double f, const double* x, const double* s, double mu,
                         double* out, int mem);
/* barrier_slope (iterate.hpp:220-236). */
int gn_ipm_barrier_slope(gn_ipm* ipm, const double* grad, const gn_iterate* it,
                         const gn_direction* d, double mu, double* out, int mem);
/* constraint_violation (iterate.hpp:238-244). */
int gn_ipm_constraint_violation(gn_ipm* ipm, const double* g, const double* s, double* out,
                                int mem);
/* kkt_error (iterate.hpp:246-298): out3 = {stat, feas, comp}. */
int gn_ipm_kkt_error(gn_ipm* ipm, const gn_iterate* it, const gn_residuals* r, double mu,
                     double* out3, int mem);
/* recover_bound_steps (condensed.hpp:187-212): reads d->dx, d->ds, writes d->dz*. */
int gn_ipm_recover_bound_steps(gn_ipm* ipm, const gn_iterate* it, const gn_residuals* r,
                               const gn_direction* d, int mem);
/* CondensedKkt::solve around the LDL^T (condensed.hpp:150-172), with the sigma_s,
 * delta_w, delta_c of the last assemble: rhs[n] = -(qx + A^T (c.qs + d.qy)) before
 * the factor solve; ds, dy from the solved dx after it. */
int gn_kkt_solve_rhs(gn_ipm* ipm, const double* qx, const double* qs, const double* qy,
                     const double* sigma_s, double delta_w, double delta_c, double* rhs, int mem);
int gn_kkt_solve_finish(gn_ipm* ipm, const double* dx, const double* qs, const double* qy,
                        const double* sigma_s, double delta_w, double delta_c, double* ds,
                        double* dy, int mem);

/* ------------------------------------------------------------ test support
 * (compute-sanitizer is unavailable on the GPU pool.)  fill = 1: write `pattern` over the
 * KKT's A and M values and the guard band allocated after each; fill = 0: out4 = {A slots
 * still holding the pattern (never written), A guard words changed (overrun), the same for
 * M}.  An assembly between the two calls must leave {0, 0, 0, 0}. */
int gn_debug_kkt_guard(gn_kkt* kkt, int fill, uint64_t pattern, int64_t* out4);

/* Page-locked host memory for host-mode outputs and inputs (cudaHostAlloc, portable):
 * GN_MEM_HOST transfers from / to it run as direct DMA, without the bounce-buffer copy
 * pageable memory needs.  The shim CondensedKkt keeps its A and M values in it. */
int gn_host_alloc(size_t bytes, void** out);
int gn_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* GRIDNLP_B200_H */
