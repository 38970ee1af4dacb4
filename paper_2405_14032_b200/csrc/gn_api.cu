// C-ABI entry points (include/gridnlp_b200.h).  Host C++: argument checking,
// memory modes, staging, error mapping.  All compute is in the kernels of
// gn_ctx.cu / gn_eval.cu / gn_kkt.cu / gn_opf_kkt.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <random>

#include "gn_ipm.cuh"
#include "gn_kkt.cuh"

using gnb::DBuf;
using gnb::Error;

namespace {

int fail(gn_error* err, int code, const char* msg, int pattern = -1, int record = -1) {
  if (err) {
    err->code = code;
    err->pattern = pattern;
    err->record = record;
    std::snprintf(err->message, sizeof err->message, "%s", msg);
  }
  return code;
}
int ok(gn_error* err) {
  if (err) {
    err->code = GN_OK;
    err->pattern = -1;
    err->record = -1;
    err->message[0] = 0;
  }
  return GN_OK;
}

#define API_TRY try {
#define API_CATCH(err)                                                   \
  }                                                                      \
  catch (const gnb::Error& e) {                                          \
    return fail(err, e.code, e.what());                                  \
  }                                                                      \
  catch (const std::exception& e) {                                      \
    return fail(err, GN_ERR_INVALID, e.what());                          \
  }

bool is_device(int mem) { return (mem & 0xf) != GN_MEM_HOST; }
bool is_async(int mem) { return (mem & 0xf) == GN_MEM_DEVICE_ASYNC; }
bool is_full(int mem) { return (mem & GN_IN_FULL) != 0; }

void set_device(int dev) { GN_CK(cudaSetDevice(dev)); }

template <class T>
std::vector<T> vec(const T* p, int64_t n, const char* what) {
  if (n > 0 && !p) throw Error(GN_ERR_INVALID, std::string("null array: ") + what);
  return n > 0 ? std::vector<T>(p, p + n) : std::vector<T>();
}

// Read and clear the latched evaluation status.
int take_status(gn_ctx* c, gn_error* err) {
  unsigned long long st = gnb::kNoFail;
  GN_CK(cudaMemcpyAsync(&st, c->status.p, sizeof st, cudaMemcpyDeviceToHost, c->stream));
  GN_CK(cudaStreamSynchronize(c->stream));
  if (st == gnb::kNoFail) return ok(err);
  GN_CK(cudaMemsetAsync(c->status.p, 0xff, sizeof st, c->stream));
  GN_CK(cudaStreamSynchronize(c->stream));
  return fail(err, GN_ERR_EVAL, "domain violation or non-finite result",
              static_cast<int>(st >> 32), static_cast<int>(st & 0xffffffffu));
}

__global__ void k_gather(int64_t n, const int32_t* __restrict__ pick,
                         const double* __restrict__ in, double* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = in[pick[k]];
}

void copy_i32(int32_t* dst, const int32_t* src, int64_t n, int mem, cudaStream_t s) {
  if (!dst || n <= 0) return;
  if (is_device(mem))
    GN_CK(cudaMemcpyAsync(dst, src, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  else
    gnb::d2h(dst, src, sizeof(int32_t) * n, s);
}

}  // namespace

extern "C" {

int gn_abi_version(void) { return GN_ABI_VERSION; }

void gn_profile_enable(int on) { gnb::profile_enable(on != 0); }
void gn_profile_reset(void) { gnb::profile_reset(); }
int gn_profile_count(void) { return gnb::profile_count(); }
const char* gn_profile_get(int i, double* total_ms, int64_t* launches) {
  return gnb::profile_get(i, total_ms, launches);
}
int64_t gn_launch_count(void) { return gnb::launch_count(); }

int gn_device_count(int32_t* n_devices) {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (n_devices) *n_devices = n;
  return n > 0 ? GN_OK : GN_ERR_CUDA;
}

// generate_load_profile (network.hpp:104-140), bit-identical: mt19937_64 and
// the top-53-bit mapping to [0,1).
int gn_load_profile(int32_t n_load, int32_t periods, double resolution_minutes, uint64_t seed,
                    double amplitude, double noise, double* scale, gn_error* err) {
  if (periods < 1) return fail(err, GN_ERR_INVALID, "load profile: need at least one period");
  if (resolution_minutes <= 0.0)
    return fail(err, GN_ERR_INVALID, "load profile: resolution must be positive");
  if (amplitude < 0.0 || amplitude >= 1.0)
    return fail(err, GN_ERR_INVALID, "load profile: amplitude must lie in [0, 1)");
  if (noise < 0.0) return fail(err, GN_ERR_INVALID, "load profile: noise must be nonnegative");
  if (n_load > 0 && !scale) return fail(err, GN_ERR_INVALID, "null scale");
  std::mt19937_64 rng(seed);
  constexpr double kTwoPi = 6.283185307179586476925286766559;
  for (int32_t t = 0; t < periods; ++t) {
    const double phase = kTwoPi * static_cast<double>(t + 1) * resolution_minutes / 1440.0;
    const double wave = 1.0 + amplitude * std::sin(phase);
    for (int32_t j = 0; j < n_load; ++j) {
      const double u01 = static_cast<double>(rng() >> 11) * 0x1.0p-53;
      const double u = 2.0 * u01 - 1.0;
      scale[static_cast<size_t>(t) * n_load + j] = std::max(0.1, wave + noise * u);
    }
  }
  return ok(err);
}

// ----------------------------------------------------------------- context
// Free a context that never left ctx_create (no dependents): its tables and its own stream.
static void ctx_discard(gn_ctx* c) {
  if (!c) return;
  cudaStream_t s = c->owned_stream;
  if (s) cudaStreamSynchronize(s);
  delete c;
  if (s) cudaStreamDestroy(s);
}

static int ctx_create(const gn_network* net, int32_t periods_total, int32_t first_period,
                      int32_t periods, const double* scale, int32_t device, gn_ctx** out,
                      gn_error* err) {
  if (!net || !out) return fail(err, GN_ERR_INVALID, "null argument");
  *out = nullptr;
  gn_ctx* c = nullptr;
  API_TRY
  const int32_t N = net->n_bus, L = net->n_line, G = net->n_gen, D = net->n_load;
  const int32_t T = periods;
  if (first_period < 0 || periods < 1 || first_period + periods > periods_total)
    throw Error(GN_ERR_INVALID, "shard: periods outside the horizon");
  if (N < 0 || L < 0 || G < 0 || D < 0) throw Error(GN_ERR_INVALID, "negative element count");
  if (net->reference_bus < 0 || net->reference_bus >= N)
    throw Error(GN_ERR_INVALID, "opf: network has no reference bus");
  if (T < 1) throw Error(GN_ERR_INVALID, "load profile: need at least one period");
  if (D > 0 && !scale) throw Error(GN_ERR_INVALID, "opf: load profile does not match network loads");
  set_device(device);
  c = new gn_ctx();
  c->device = device;
  c->bus_vmin = vec(net->bus_vmin, N, "bus_vmin");
  c->bus_vmax = vec(net->bus_vmax, N, "bus_vmax");
  c->vm_start = vec(net->vm_start, N, "vm_start");
  c->va_start = vec(net->va_start, N, "va_start");
  c->line_from = vec(net->line_from, L, "line_from");
  c->line_to = vec(net->line_to, L, "line_to");
  c->line_g = vec(net->line_g, L, "line_g");
  c->line_b = vec(net->line_b, L, "line_b");
  c->line_smax = vec(net->line_smax, L, "line_smax");
  c->line_amin = vec(net->line_amin, L, "line_amin");
  c->line_amax = vec(net->line_amax, L, "line_amax");
  c->gen_bus = vec(net->gen_bus, G, "gen_bus");
  c->gen_pmin = vec(net->gen_pmin, G, "gen_pmin");
  c->gen_pmax = vec(net->gen_pmax, G, "gen_pmax");
  c->gen_qmin = vec(net->gen_qmin, G, "gen_qmin");
  c->gen_qmax = vec(net->gen_qmax, G, "gen_qmax");
  c->gen_ramp = vec(net->gen_ramp, G, "gen_ramp");
  c->gen_c2 = vec(net->gen_c2, G, "gen_c2");
  c->gen_c1 = vec(net->gen_c1, G, "gen_c1");
  c->gen_c0 = vec(net->gen_c0, G, "gen_c0");
  c->gen_pstart = vec(net->gen_pstart, G, "gen_pstart");
  c->gen_qstart = vec(net->gen_qstart, G, "gen_qstart");
  std::vector<int32_t> load_bus = vec(net->load_bus, D, "load_bus");
  std::vector<double> load_p = vec(net->load_p, D, "load_p"), load_q = vec(net->load_q, D, "load_q");

  // Reference validation (PatternModel::add_* throws on these; opf.hpp:105-108).
  for (int32_t l = 0; l < L; ++l) {
    const int32_t f = c->line_from[l], t = c->line_to[l];
    if (f < 0 || f >= N || t < 0 || t >= N) throw Error(GN_ERR_INVALID, "line references unknown bus");
    if (c->line_amin[l] > c->line_amax[l])
      throw Error(GN_ERR_INVALID, "constraint block angle: lower above upper");
  }
  for (int32_t g = 0; g < G; ++g) {
    if (c->gen_bus[g] < 0 || c->gen_bus[g] >= N) throw Error(GN_ERR_INVALID, "generator references unknown bus");
    if (c->gen_pmin[g] > c->gen_pmax[g]) throw Error(GN_ERR_INVALID, "variable block pg: lower above upper");
    if (c->gen_qmin[g] > c->gen_qmax[g]) throw Error(GN_ERR_INVALID, "variable block qg: lower above upper");
  }
  for (int32_t n = 0; n < N; ++n)
    if (c->bus_vmin[n] > c->bus_vmax[n]) throw Error(GN_ERR_INVALID, "variable block v: lower above upper");
  for (int32_t j = 0; j < D; ++j)
    if (load_bus[j] < 0 || load_bus[j] >= N) throw Error(GN_ERR_INVALID, "load references unknown bus");
  const double inf = std::numeric_limits<double>::infinity();
  for (int32_t l = 0; l < L; ++l)
    if (c->line_smax[l] < inf) c->thermal_lines.push_back(l);
  if (periods_total >= 2)  // ramp rows exist when the whole horizon has >= 2 periods
    for (int32_t g = 0; g < G; ++g)
      if (c->gen_ramp[g] < inf) {
        if (-c->gen_ramp[g] > c->gen_ramp[g])
          throw Error(GN_ERR_INVALID, "constraint block ramp: lower above upper");
        c->ramp_gens.push_back(g);
      }
  const int32_t LT = static_cast<int32_t>(c->thermal_lines.size());
  const int32_t GR = static_cast<int32_t>(c->ramp_gens.size());
  c->d = gnb::make_dims(T, N, L, G, D, LT, GR, net->reference_bus, first_period, periods_total);

  GN_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  c->owned_stream = c->stream;
  cudaStream_t s = c->stream;

  // SoA tables
  std::vector<int32_t> l_therm(L, -1);
  for (int32_t k = 0; k < LT; ++k) l_therm[c->thermal_lines[k]] = k;
  c->lf.upload(c->line_from.data(), L, s);
  c->lt.upload(c->line_to.data(), L, s);
  c->lg.upload(c->line_g.data(), L, s);
  c->lb.upload(c->line_b.data(), L, s);
  c->l_therm.upload(l_therm.data(), L, s);
  c->th_line.upload(c->thermal_lines.data(), LT, s);
  c->gbus.upload(c->gen_bus.data(), G, s);
  c->c2.upload(c->gen_c2.data(), G, s);
  c->c1.upload(c->gen_c1.data(), G, s);
  c->c0.upload(c->gen_c0.data(), G, s);
  c->ramp_gen.upload(c->ramp_gens.data(), GR, s);
  // demand pd(t,j) = load.p * scale[t*D+j] (network.hpp:166-171), entity-major
  {
    std::vector<double> pd(static_cast<size_t>(D) * T), qd(static_cast<size_t>(D) * T);
    for (int32_t j = 0; j < D; ++j)
      for (int32_t t = 0; t < T; ++t) {
        const double sc = scale[static_cast<size_t>(t) * D + j];
        pd[static_cast<size_t>(j) * T + t] = load_p[j] * sc;
        qd[static_cast<size_t>(j) * T + t] = load_q[j] * sc;
      }
    c->pd.upload(pd.data(), pd.size(), s);
    c->qd.upload(qd.data(), qd.size(), s);
    GN_CK(cudaStreamSynchronize(s));
  }
  // bus incidence in the reference's accumulation order
  {
    std::vector<std::vector<int32_t>> bl(N), bg(N), bd(N);
    for (int32_t l = 0; l < L; ++l) {
      bl[c->line_to[l]].push_back(l << 1);          // to-record, s = +1
      bl[c->line_from[l]].push_back((l << 1) | 1);  // from-record, s = -1
    }
    for (int32_t g = 0; g < G; ++g) bg[c->gen_bus[g]].push_back(g);
    for (int32_t j = 0; j < D; ++j) bd[load_bus[j]].push_back(j);
    auto flat = [&](std::vector<std::vector<int32_t>>& v, DBuf<int32_t>& ptr, DBuf<int32_t>& idx) {
      std::vector<int32_t> p(N + 1, 0), x;
      for (int32_t n = 0; n < N; ++n) {
        p[n + 1] = p[n] + static_cast<int32_t>(v[n].size());
        x.insert(x.end(), v[n].begin(), v[n].end());
      }
      ptr.upload(p.data(), p.size(), s);
      idx.upload(x.data(), x.size(), s);
      GN_CK(cudaStreamSynchronize(s));
    };
    flat(bl, c->bl_ptr, c->bl);
    flat(bg, c->bg_ptr, c->bg);
    flat(bd, c->bd_ptr, c->bd);
  }
  c->status.alloc(1);
  GN_CK(cudaMemsetAsync(c->status.p, 0xff, sizeof(unsigned long long), s));
  c->fpart.alloc(gnb::fpart_size(c->d));
  GN_CK(cudaMemsetAsync(c->fpart.p, 0, sizeof(double) * gnb::fpart_size(c->d), s));
  GN_CK(cudaStreamSynchronize(s));
  *out = c;
  return ok(err);
  }
  catch (const gnb::Error& e) {
    ctx_discard(c);
    return fail(err, e.code, e.what());
  }
  catch (const std::exception& e) {
    ctx_discard(c);
    return fail(err, GN_ERR_INVALID, e.what());
  }
}

int gn_ctx_create(const gn_network* net, int32_t periods, const double* scale, int32_t device,
                  gn_ctx** out, gn_error* err) {
  return ctx_create(net, periods, 0, periods, scale, device, out, err);
}

int gn_ctx_create_shard(const gn_network* net, int32_t periods_total, int32_t first_period,
                        int32_t periods, const double* scale, int32_t device, gn_ctx** out,
                        gn_error* err) {
  return ctx_create(net, periods_total, first_period, periods, scale, device, out, err);
}

int gn_ctx_shard_info(gn_ctx* c, int64_t* info, int32_t* ramp_gens) {
  if (!c || !info) return GN_ERR_INVALID;
  const auto& d = c->d;
  const int64_t v[12] = {d.t0, d.T_total, d.prev, d.next, d.GR, d.n_base, d.gh_prev, d.gh_next,
                         d.ramp0, d.R, d.s_lo, c->lifted ? (int64_t)c->n_free - (d.next ? d.GR : 0) : -1};
  for (int i = 0; i < 12; ++i) info[i] = v[i];
  if (ramp_gens)
    for (int32_t k = 0; k < d.GR; ++k) ramp_gens[k] = c->ramp_gens[k];
  return GN_OK;
}

// ------------------------------------------------------- published contexts
// A context published with gn_ctx_publish lets gn_kkt_create recognise its lifted
// structure: the reference's IpmSolver builds its CondensedKkt from plain COO arrays
// (solver.hpp:139-141), and the match gives that KKT the OPF-specialised kernels.
}  // extern "C"
namespace {
std::mutex g_pub_mu;
std::vector<gn_ctx*> g_published;
void unpublish(gn_ctx* c) {
  std::lock_guard<std::mutex> lk(g_pub_mu);
  g_published.erase(std::remove(g_published.begin(), g_published.end(), c), g_published.end());
}
}  // namespace

gn_ctx* gnb::find_published(int device, int32_t n, int32_t m, int64_t nj, const int32_t* jr,
                            const int32_t* jc, int64_t nh, const int32_t* hr, const int32_t* hc,
                            cudaStream_t s) {
  std::vector<gn_ctx*> cands;
  {
    std::lock_guard<std::mutex> lk(g_pub_mu);
    for (gn_ctx* c : g_published)
      if (!c->closed && c->device == device && c->lifted && c->n_free == n && c->d.m == m &&
          c->nj_l == nj && c->nh_l == nh)
        cands.push_back(c);
  }
  if (cands.empty()) return nullptr;
  DBuf<int32_t> diff;
  diff.alloc(1);
  for (gn_ctx* c : cands) {
    GN_CK(cudaMemsetAsync(diff.p, 0, 4, s));
    gnb::count_diff(jr, c->jr_l.p, nj, diff.p, s);
    gnb::count_diff(jc, c->jc_l.p, nj, diff.p, s);
    gnb::count_diff(hr, c->hr_l.p, nh, diff.p, s);
    gnb::count_diff(hc, c->hc_l.p, nh, diff.p, s);
    int32_t h = 1;
    GN_CK(cudaMemcpyAsync(&h, diff.p, 4, cudaMemcpyDeviceToHost, s));
    GN_CK(cudaStreamSynchronize(s));
    if (h == 0) return c;
  }
  return nullptr;
}

extern "C" {

int gn_ctx_publish(gn_ctx* c, int on) {
  if (!c) return GN_ERR_INVALID;
  API_TRY
  set_device(c->device);
  if (on && !c->lifted) {  // the structure to match is the lifted one (lifted.hpp:73-93)
    gnb::build_lifted(c);
    c->relax = 0.0;
  }
  unpublish(c);
  if (on) {
    std::lock_guard<std::mutex> lk(g_pub_mu);
    g_published.push_back(c);
  }
  return GN_OK;
  API_CATCH(nullptr)
}

// Objects built on another (a KKT on a context, an IPM on a KKT) hold a reference: a
// destroy call on an object still referenced only marks it closed, and the last
// dependent's destroy frees it -- destroy calls may come in any order (e.g. from a
// garbage collector) without a dependent ever touching a freed stream or table.
static void ctx_free(gn_ctx* c) {
  unpublish(c);
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaStream_t s = c->owned_stream;  // the caller's stream (set_stream) is never destroyed
  delete c;
  if (s) cudaStreamDestroy(s);
}

}  // extern "C"
void gnb::ctx_unref(gn_ctx* c) {
  if (c && --c->refs == 0 && c->closed) ctx_free(c);
}
extern "C" {

int gn_ctx_destroy(gn_ctx* c) {
  if (!c) return GN_OK;
  unpublish(c);  // no new KKT may match it; live ones keep their reference
  c->closed = true;
  if (c->refs == 0) ctx_free(c);
  return GN_OK;
}

int gn_ctx_set_stream(gn_ctx* c, void* stream) {
  if (!c) return GN_ERR_INVALID;
  API_TRY
  set_device(c->device);
  if ((stream ? static_cast<cudaStream_t>(stream) : c->owned_stream) == c->stream) return GN_OK;
  GN_CK(cudaStreamSynchronize(c->stream));
  // the context's own stream stays alive until gn_ctx_destroy: a KKT created on it
  // may still reference it
  c->stream = stream ? static_cast<cudaStream_t>(stream) : c->owned_stream;
  c->own_stream = c->stream == c->owned_stream;
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_ctx_get_stream(gn_ctx* c, void** stream) {
  if (!c || !stream) return GN_ERR_INVALID;
  *stream = c->stream;
  return GN_OK;
}

int gn_ctx_status(gn_ctx* c, gn_error* err) {
  if (!c) return fail(err, GN_ERR_INVALID, "null context");
  API_TRY
  set_device(c->device);
  return take_status(c, err);
  API_CATCH(err)
}

int gn_ctx_sizes(gn_ctx* c, gn_sizes* o) {
  if (!c || !o) return GN_ERR_INVALID;
  const auto& d = c->d;
  o->n_vars = d.n;
  o->n_cons = d.m;
  o->jac_nnz = d.nj;
  o->hess_nnz = d.nh;
  o->n_thermal = d.LT;
  o->n_ramp_gens = d.GR;
  o->periods = d.T;
  o->n_free = c->lifted ? c->n_free : -1;
  o->jac_nnz_lifted = c->lifted ? c->nj_l : -1;
  o->hess_nnz_lifted = c->lifted ? c->nh_l : -1;
  return GN_OK;
}

int gn_ctx_bounds(gn_ctx* c, double* xl, double* xu, double* xs, double* rl, double* ru) {
  if (!c) return GN_ERR_INVALID;
  API_TRY
  gnb::host_bounds(c, xl, xu, xs, rl, ru);
  return GN_OK;
  API_CATCH(nullptr)
}

static int structure(gn_ctx* c, bool jac, int32_t* rows, int32_t* cols, int mem) {
  if (!c) return GN_ERR_INVALID;
  API_TRY
  set_device(c->device);
  const auto& d = c->d;
  DBuf<int32_t> r, k;  // only the requested structure is built
  const int64_t n = jac ? d.nj : d.nh;
  r.alloc(n + 1);
  k.alloc(n + 1);
  if (jac) gnb::build_structure(c, r.p, k.p, nullptr, nullptr);
  else gnb::build_structure(c, nullptr, nullptr, r.p, k.p);
  copy_i32(rows, r.p, n, mem, c->stream);
  copy_i32(cols, k.p, n, mem, c->stream);
  GN_CK(cudaStreamSynchronize(c->stream));
  return GN_OK;
  API_CATCH(nullptr)
}
int gn_jac_structure(gn_ctx* c, int32_t* rows, int32_t* cols, int mem) {
  return structure(c, true, rows, cols, mem);
}
int gn_hess_structure(gn_ctx* c, int32_t* rows, int32_t* cols, int mem) {
  return structure(c, false, rows, cols, mem);
}

// ---------------------------------------------------------------- callbacks
static int eval(gn_ctx* c, int mode, const double* x, const double* w, double ow, double* out,
                int mem, gn_error* err) {
  if (!c) return fail(err, GN_ERR_INVALID, "null context");
  if (!x || !out || (mode == gnb::EV_H && !w)) return fail(err, GN_ERR_INVALID, "null array");
  API_TRY
  set_device(c->device);
  const auto& d = c->d;
  cudaStream_t s = c->stream;
  const int64_t nout = mode == gnb::EV_F ? 1 : mode == gnb::EV_GRAD ? d.n
                       : mode == gnb::EV_G ? d.m : mode == gnb::EV_J ? d.nj : d.nh;
  const double* dx = x;
  const double* dw = w;
  double* dout = out;
  if (!is_device(mem)) {
    c->sx.upload(x, d.n, s);
    dx = c->sx.p;
    if (mode == gnb::EV_H) {
      c->sw.upload(w, d.m, s);
      dw = c->sw.p;
    }
    if (c->sout.n < static_cast<size_t>(nout)) c->sout.alloc(nout);
    dout = c->sout.p;
  }
  if (!is_async(mem))
    GN_CK(cudaMemsetAsync(c->status.p, 0xff, sizeof(unsigned long long), s));
  gnb::launch_eval(mode, d, c->net(), dx, dw, ow, dout, c->fpart.p, c->status.p, s);
  if (is_async(mem)) return ok(err);
  if (!is_device(mem))
    gnb::d2h(out, dout, sizeof(double) * nout, s);
  return take_status(c, err);
  API_CATCH(err)
}

int gn_eval_f(gn_ctx* c, const double* x, double* out, int mem, gn_error* err) {
  return eval(c, gnb::EV_F, x, nullptr, 0.0, out, mem, err);
}
int gn_eval_grad(gn_ctx* c, const double* x, double* out, int mem, gn_error* err) {
  return eval(c, gnb::EV_GRAD, x, nullptr, 0.0, out, mem, err);
}
int gn_eval_g(gn_ctx* c, const double* x, double* out, int mem, gn_error* err) {
  return eval(c, gnb::EV_G, x, nullptr, 0.0, out, mem, err);
}
int gn_eval_jac(gn_ctx* c, const double* x, double* out, int mem, gn_error* err) {
  return eval(c, gnb::EV_J, x, nullptr, 0.0, out, mem, err);
}
int gn_eval_hess(gn_ctx* c, const double* x, const double* w, double ow, double* out, int mem,
                 gn_error* err) {
  return eval(c, gnb::EV_H, x, w, ow, out, mem, err);
}

// One IPM iteration's callbacks (solver.hpp:157-158, 202: eval_f, eval_grad, eval_g,
// eval_jac, then eval_hess at the same x) in one kernel launch; outputs bit-identical to
// the five gn_eval_* calls, one status word for all five.
int gn_eval_all(gn_ctx* c, const double* x, const double* w, double ow, double* f,
                double* grad, double* g, double* jac, double* hess, int mem, gn_error* err) {
  if (!c) return fail(err, GN_ERR_INVALID, "null context");
  if (!x || !w || !f || !grad || !g || !jac || !hess) return fail(err, GN_ERR_INVALID, "null array");
  API_TRY
  set_device(c->device);
  const auto& d = c->d;
  cudaStream_t s = c->stream;
  const double *dx = x, *dw = w;
  double *df = f, *dgr = grad, *dg = g, *dj = jac, *dh = hess;
  if (!is_device(mem)) {
    c->sx.upload(x, d.n, s);
    c->sw.upload(w, d.m, s);
    dx = c->sx.p;
    dw = c->sw.p;
    const size_t need = static_cast<size_t>(1 + d.n + d.m + d.nj + d.nh);
    if (c->sout.n < need) c->sout.alloc(need);
    df = c->sout.p;
    dgr = df + 1;
    dg = dgr + d.n;
    dj = dg + d.m;
    dh = dj + d.nj;
  }
  if (!is_async(mem))
    GN_CK(cudaMemsetAsync(c->status.p, 0xff, sizeof(unsigned long long), s));
  gnb::launch_eval_all(d, c->net(), dx, dw, ow, df, dgr, dg, dj, dh, c->fpart.p, c->status.p, s);
  if (is_async(mem)) return ok(err);
  if (!is_device(mem)) {
    gnb::d2h(f, df, sizeof(double), s);
    gnb::d2h(grad, dgr, sizeof(double) * d.n, s);
    gnb::d2h(g, dg, sizeof(double) * d.m, s);
    gnb::d2h(jac, dj, sizeof(double) * d.nj, s);
    gnb::d2h(hess, dh, sizeof(double) * d.nh, s);
  }
  return take_status(c, err);
  API_CATCH(err)
}

// Line-search trial point (solver.hpp:267-304): the objective and
// the constraint values only -- no derivative kernels -- under one status word.
int gn_eval_fg(gn_ctx* c, const double* x, double* f, double* g, int mem, gn_error* err) {
  if (!c) return fail(err, GN_ERR_INVALID, "null context");
  if (!x || !f || !g) return fail(err, GN_ERR_INVALID, "null array");
  API_TRY
  set_device(c->device);
  const auto& d = c->d;
  cudaStream_t s = c->stream;
  const double* dx = x;
  double *df = f, *dg = g;
  if (!is_device(mem)) {
    c->sx.upload(x, d.n, s);
    dx = c->sx.p;
    if (c->sout.n < static_cast<size_t>(d.m) + 1) c->sout.alloc(static_cast<size_t>(d.m) + 1);
    dg = c->sout.p;
    df = c->sout.p + d.m;
  }
  if (!is_async(mem))
    GN_CK(cudaMemsetAsync(c->status.p, 0xff, sizeof(unsigned long long), s));
  gnb::launch_eval(gnb::EV_FG, d, c->net(), dx, nullptr, 0.0, dg, c->fpart.p, c->status.p, s, df);
  if (is_async(mem)) return ok(err);
  if (!is_device(mem)) {
    gnb::d2h(g, dg, sizeof(double) * d.m, s);
    gnb::d2h(f, df, sizeof(double), s);
  }
  return take_status(c, err);
  API_CATCH(err)
}

// ------------------------------------------------------------------- lifted
int gn_lifted_create(gn_ctx* c, double relax, gn_error* err) {
  if (!c) return fail(err, GN_ERR_INVALID, "null context");
  API_TRY
  set_device(c->device);
  // the filter does not depend on relax (only the slack boxes do): built once, so KKTs
  // already built on this context's lifted arrays (gn_ctx_publish) keep them
  if (!c->lifted) gnb::build_lifted(c);
  c->relax = relax;
  return ok(err);
  API_CATCH(err)
}

int gn_lifted_structure(gn_ctx* c, int32_t* free_to_full, int32_t* jr, int32_t* jc,
                        int32_t* jpick, int32_t* hr, int32_t* hc, int32_t* hpick, double* sl,
                        double* su, int mem) {
  if (!c || !c->lifted) return GN_ERR_INVALID;
  API_TRY
  set_device(c->device);
  cudaStream_t s = c->stream;
  copy_i32(free_to_full, c->full_of_free.p, c->n_free, mem, s);
  copy_i32(jr, c->jr_l.p, c->nj_l, mem, s);
  copy_i32(jc, c->jc_l.p, c->nj_l, mem, s);
  copy_i32(jpick, c->jpick.p, c->nj_l, mem, s);
  copy_i32(hr, c->hr_l.p, c->nh_l, mem, s);
  copy_i32(hc, c->hc_l.p, c->nh_l, mem, s);
  copy_i32(hpick, c->hpick.p, c->nh_l, mem, s);
  GN_CK(cudaStreamSynchronize(s));
  if (sl || su) {  // slack boxes (lifted.hpp:160-176), host
    const int32_t m = c->d.m;
    std::vector<double> rl(m), ru(m);
    gnb::host_bounds(c, nullptr, nullptr, nullptr, rl.data(), ru.data());
    for (int32_t i = 0; i < m; ++i) {
      const double lo = rl[i], hi = ru[i];
      double a = lo, b = hi;
      if (lo == hi) {
        const double width = c->relax * std::max(1.0, std::abs(lo));
        a = lo - width;
        b = hi + width;
      }
      if (sl) sl[i] = a;
      if (su) su[i] = b;
    }
  }
  return GN_OK;
  API_CATCH(nullptr)
}

static int lifted_gather(gn_ctx* c, bool jac, const double* in, double* out, int mem) {
  if (!c || !c->lifted || !in || !out) return GN_ERR_INVALID;
  API_TRY
  set_device(c->device);
  cudaStream_t s = c->stream;
  const int64_t nf = jac ? c->d.nj : c->d.nh, nl = jac ? c->nj_l : c->nh_l;
  const int32_t* pick = jac ? c->jpick.p : c->hpick.p;
  const double* din = in;
  double* dout = out;
  DBuf<double> a, b;
  if (!is_device(mem)) {
    a.upload(in, nf, s);
    b.alloc(nl + 1);
    din = a.p;
    dout = b.p;
  }
  if (nl) {
    k_gather<<<(unsigned)((nl + 255) / 256), 256, 0, s>>>(nl, pick, din, dout);
    gnb::count_launch();
  }
  if (!is_device(mem)) gnb::d2h(out, dout, sizeof(double) * nl, s);
  if (!is_async(mem)) GN_CK(cudaStreamSynchronize(s));
  return GN_OK;
  API_CATCH(nullptr)
}
int gn_lifted_gather_jac(gn_ctx* c, const double* in, double* out, int mem) {
  return lifted_gather(c, true, in, out, mem);
}
int gn_lifted_gather_hess(gn_ctx* c, const double* in, double* out, int mem) {
  return lifted_gather(c, false, in, out, mem);
}

// x_full[full_of_free[k]] = x_free[k]: LiftedProblem::stage (lifted.hpp:165-168) on the device
__global__ void k_lift_stage(int64_t n, const int32_t* __restrict__ full_of_free,
                             const double* __restrict__ x_free, double* __restrict__ x_full) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) x_full[full_of_free[k]] = x_free[k];
}

// LiftedProblem::eval_* (lifted.hpp:128-159) in one call on the device: the free-variable
// point is staged into the full space (fixed entries at their pinned values, the
// reference's fixed_value_), the full-space callback runs, and the lifted outputs are
// gathered on the device -- only lifted-size arrays cross PCIe in the host modes.
static int lifted_eval(gn_ctx* c, int mode, const double* x, const double* w, double ow,
                       double* out, double* fout, int mem, gn_error* err) {
  if (!c) return fail(err, GN_ERR_INVALID, "null context");
  if (!c->lifted) return fail(err, GN_ERR_INVALID, "gn_lifted_create must run first");
  if (!x || !out || (mode == gnb::EV_H && !w) || (mode == gnb::EV_FG && !fout))
    return fail(err, GN_ERR_INVALID, "null array");
  if (c->d.n != c->d.n_base)  // ghost set-points hold halo values the staging cannot know
    return fail(err, GN_ERR_UNSUPPORTED,
                "lifted evaluation of a period shard: use the full-space calls with the halo");
  API_TRY
  set_device(c->device);
  const auto& d = c->d;
  cudaStream_t s = c->stream;
  if (!c->lx_ready) {  // fixed_value_: xl where xl == xu (lifted.hpp:35-45), else overwritten
    std::vector<double> xl(d.n), xu(d.n);
    gnb::host_bounds(c, xl.data(), xu.data(), nullptr, nullptr, nullptr);
    for (int64_t i = 0; i < d.n; ++i) xl[i] = xl[i] == xu[i] ? xl[i] : 0.0;
    c->lx.upload(xl.data(), d.n, s);
    c->lx_ready = true;
  }
  const int64_t nf = c->n_free;
  const double* dxf = x;
  if (!is_device(mem)) {
    c->lxin.upload(x, nf, s);
    dxf = c->lxin.p;
  }
  if (nf) {
    k_lift_stage<<<(unsigned)((nf + 255) / 256), 256, 0, s>>>(nf, c->full_of_free.p, dxf, c->lx.p);
    gnb::count_launch();
  }
  const double* dw = w;
  if (mode == gnb::EV_H && !is_device(mem)) {
    c->sw.upload(w, d.m, s);
    dw = c->sw.p;
  }
  // full-space output; f and g are not lifted (rows keep their numbering)
  const bool gathered = mode == gnb::EV_GRAD || mode == gnb::EV_J || mode == gnb::EV_H;
  const int64_t nfull = mode == gnb::EV_F ? 1 : mode == gnb::EV_GRAD ? d.n
                        : mode == gnb::EV_J ? d.nj : mode == gnb::EV_H ? d.nh : d.m + 1;
  const int64_t nout = mode == gnb::EV_GRAD ? nf : mode == gnb::EV_J ? c->nj_l
                       : mode == gnb::EV_H ? c->nh_l : mode == gnb::EV_F ? 1 : d.m;
  double* dfull = out;
  if (gathered || !is_device(mem)) {
    if (c->sout.n < static_cast<size_t>(nfull)) c->sout.alloc(nfull);
    dfull = c->sout.p;
  }
  double* df = mode == gnb::EV_FG ? (is_device(mem) ? fout : c->sout.p + d.m) : nullptr;
  if (!is_async(mem))
    GN_CK(cudaMemsetAsync(c->status.p, 0xff, sizeof(unsigned long long), s));
  gnb::launch_eval(mode, d, c->net(), c->lx.p, dw, ow, dfull, c->fpart.p, c->status.p, s, df);
  double* dout = dfull;
  if (gathered) {
    const int32_t* pick = mode == gnb::EV_GRAD ? c->full_of_free.p
                          : mode == gnb::EV_J ? c->jpick.p : c->hpick.p;
    dout = out;
    if (!is_device(mem)) {
      if (c->lout.n < static_cast<size_t>(nout) + 1) c->lout.alloc(nout + 1);
      dout = c->lout.p;
    }
    if (nout) {
      k_gather<<<(unsigned)((nout + 255) / 256), 256, 0, s>>>(nout, pick, dfull, dout);
      gnb::count_launch();
    }
  }
  if (is_async(mem)) return ok(err);
  if (!is_device(mem)) {
    gnb::d2h(out, dout, sizeof(double) * nout, s);
    if (mode == gnb::EV_FG) gnb::d2h(fout, df, sizeof(double), s);
  }
  return take_status(c, err);
  API_CATCH(err)
}

int gn_lifted_eval_f(gn_ctx* c, const double* x, double* out, int mem, gn_error* err) {
  return lifted_eval(c, gnb::EV_F, x, nullptr, 0.0, out, nullptr, mem, err);
}
int gn_lifted_eval_grad(gn_ctx* c, const double* x, double* out, int mem, gn_error* err) {
  return lifted_eval(c, gnb::EV_GRAD, x, nullptr, 0.0, out, nullptr, mem, err);
}
int gn_lifted_eval_g(gn_ctx* c, const double* x, double* out, int mem, gn_error* err) {
  return lifted_eval(c, gnb::EV_G, x, nullptr, 0.0, out, nullptr, mem, err);
}
int gn_lifted_eval_jac(gn_ctx* c, const double* x, double* out, int mem, gn_error* err) {
  return lifted_eval(c, gnb::EV_J, x, nullptr, 0.0, out, nullptr, mem, err);
}
int gn_lifted_eval_hess(gn_ctx* c, const double* x, const double* w, double ow, double* out,
                        int mem, gn_error* err) {
  return lifted_eval(c, gnb::EV_H, x, w, ow, out, nullptr, mem, err);
}
int gn_lifted_eval_fg(gn_ctx* c, const double* x, double* f, double* g, int mem,
                      gn_error* err) {
  return lifted_eval(c, gnb::EV_FG, x, nullptr, 0.0, g, f, mem, err);
}

// --------------------------------------------------------------------- KKT
int gn_kkt_create(int32_t n, int32_t m, int64_t nj, const int32_t* jr, const int32_t* jc,
                  int64_t nh, const int32_t* hr, const int32_t* hc, int32_t device,
                  gn_kkt** out, gn_error* err) {
  if (!out) return fail(err, GN_ERR_INVALID, "null argument");
  *out = nullptr;
  if (n < 0 || m < 0 || nj < 0 || nh < 0) return fail(err, GN_ERR_INVALID, "negative size");
  if ((nj && (!jr || !jc)) || (nh && (!hr || !hc))) return fail(err, GN_ERR_INVALID, "null array");
  gn_kkt* K = nullptr;
  API_TRY
  set_device(device);
  K = new gn_kkt();
  K->device = device;
  K->n = n; K->m = m; K->nj = nj; K->nh = nh;
  GN_CK(cudaStreamCreateWithFlags(&K->stream, cudaStreamNonBlocking));
  K->own_stream = true;
  K->owned_stream = K->stream;
  DBuf<int32_t> djr, djc, dhr, dhc;
  djr.upload(jr, nj, K->stream); djc.upload(jc, nj, K->stream);
  dhr.upload(hr, nh, K->stream); dhc.upload(hc, nh, K->stream);
  gnb::kkt_build(K, djr.p, djc.p, dhr.p, dhc.p);
  // the lifted structure of a published OPF context: same KKT, specialised kernels
  if (gn_ctx* c = gnb::find_published(device, n, m, nj, djr.p, djc.p, nh, dhr.p, dhc.p,
                                      K->stream)) {
    const char* env = std::getenv("GRIDNLP_B200_GENERIC_KKT");
    K->ctx = c;
    ++c->refs;
    if (!(env && env[0] == '1')) gnb::opf_kkt_prepare(K);
  }
  *out = K;
  return ok(err);
  }
  catch (const gnb::Error& e) {
    if (K) gn_kkt_destroy(K);
    return fail(err, e.code, e.what());
  }
  catch (const std::exception& e) {
    if (K) gn_kkt_destroy(K);
    return fail(err, GN_ERR_INVALID, e.what());
  }
}

int gn_kkt_create_lifted(gn_ctx* c, gn_kkt** out, gn_error* err) {
  if (!c || !out) return fail(err, GN_ERR_INVALID, "null argument");
  if (!c->lifted) return fail(err, GN_ERR_INVALID, "gn_lifted_create must run first");
  *out = nullptr;
  gn_kkt* K = nullptr;
  API_TRY
  set_device(c->device);
  K = new gn_kkt();
  K->device = c->device;
  K->ctx = c;
  ++c->refs;
  K->stream = c->stream;
  K->own_stream = false;
  K->n = c->n_free; K->m = c->d.m; K->nj = c->nj_l; K->nh = c->nh_l;
  gnb::kkt_build(K, c->jr_l.p, c->jc_l.p, c->hr_l.p, c->hc_l.p);
  const char* env = std::getenv("GRIDNLP_B200_GENERIC_KKT");
  if (!(env && env[0] == '1')) gnb::opf_kkt_prepare(K);
  *out = K;
  return ok(err);
  }
  catch (const gnb::Error& e) {
    if (K) gn_kkt_destroy(K);
    return fail(err, e.code, e.what());
  }
  catch (const std::exception& e) {
    if (K) gn_kkt_destroy(K);
    return fail(err, GN_ERR_INVALID, e.what());
  }
}

static void kkt_free(gn_kkt* K) {
  cudaSetDevice(K->device);
  if (K->stream) cudaStreamSynchronize(K->stream);
  if (K->vstream) {
    cudaStreamSynchronize(K->vstream);
    cudaStreamDestroy(K->vstream);
  }
  if (K->vstart) cudaEventDestroy(K->vstart);
  if (K->vdone) cudaEventDestroy(K->vdone);
  cudaStream_t s = K->owned_stream;
  gn_ctx* c = K->ctx;
  gnb::opf_kkt_free(K);
  delete K;
  if (s) cudaStreamDestroy(s);
  if (c && --c->refs == 0 && c->closed) ctx_free(c);
}

int gn_kkt_destroy(gn_kkt* K) {
  if (!K) return GN_OK;
  K->closed = true;
  if (K->refs == 0) kkt_free(K);
  return GN_OK;
}

int gn_kkt_set_stream(gn_kkt* K, void* stream) {
  if (!K) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  // NULL: back to the object's own stream -- a KKT built on a context has none of its
  // own and returns to the context's (never the legacy default stream)
  cudaStream_t own = K->owned_stream ? K->owned_stream : K->ctx->owned_stream;
  cudaStream_t want = stream ? static_cast<cudaStream_t>(stream) : own;
  if (want == K->stream) return GN_OK;
  GN_CK(cudaStreamSynchronize(K->stream));
  K->stream = want;
  K->own_stream = K->stream == own;
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_dims(gn_kkt* K, int64_t* dims) {
  if (!K || !dims) return GN_ERR_INVALID;
  dims[0] = K->n; dims[1] = K->annz; dims[2] = K->mnnz; dims[3] = K->npair;
  dims[4] = K->nj; dims[5] = K->nh; dims[6] = K->m;
  dims[7] = gnb::opf_kkt_ready(K) ? 1 : 0;
  dims[8] = gnb::opf_fused_ready(K) ? 1 : 0;
  return GN_OK;
}

int gn_kkt_structure(gn_kkt* K, int32_t* rowptr, int32_t* colidx, int32_t* colptr,
                     int32_t* rowidx, int mem) {
  if (!K) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  copy_i32(rowptr, K->A.ptr.p, (int64_t)K->m + 1, mem, K->stream);
  copy_i32(colidx, K->A.idx.p, K->annz, mem, K->stream);
  copy_i32(colptr, K->M.ptr.p, (int64_t)K->n + 1, mem, K->stream);
  copy_i32(rowidx, K->M.idx.p, K->mnnz, mem, K->stream);
  GN_CK(cudaStreamSynchronize(K->stream));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_slots(gn_kkt* K, int32_t* js, int32_t* hs, int32_t* ps, int32_t* ds, int mem) {
  if (!K) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  copy_i32(js, K->A.slot.p, K->nj, mem, K->stream);
  copy_i32(hs, K->M.slot.p, K->nh, mem, K->stream);
  copy_i32(ps, K->M.slot.p + K->nh, K->npair, mem, K->stream);
  copy_i32(ds, K->M.slot.p + K->nh + K->npair, K->n, mem, K->stream);
  GN_CK(cudaStreamSynchronize(K->stream));
  return GN_OK;
  API_CATCH(nullptr)
}

// A and M may still be read back on the side stream (gn_kkt_values_start): a kernel that
// writes one of them first waits for that copy on the device (no host synchronisation).
// Called after the host-mode uploads, so those overlap the read-back.
static void order_after_values(gn_kkt* K, bool writes_a, bool writes_m) {
  if (!((writes_a && K->vpend_a) || (writes_m && K->vpend_m))) return;
  GN_CK(cudaStreamWaitEvent(K->stream, K->vdone, 0));
  K->vpend_a = K->vpend_m = false;
}

int gn_kkt_set_jacobian(gn_kkt* K, const double* jv, int mem) {
  if (!K || !jv) return GN_ERR_INVALID;
  if (is_full(mem) && !K->ctx) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  const double* dj = jv;
  if (!is_device(mem)) {
    const int64_t n = is_full(mem) ? K->ctx->d.nj : K->nj;
    K->sj.upload(jv, n, K->stream);
    dj = K->sj.p;
  }
  order_after_values(K, true, false);
  gnb::kkt_set_jacobian(K, dj, is_full(mem));
  if (!is_async(mem)) GN_CK(cudaStreamSynchronize(K->stream));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_assemble(gn_kkt* K, const double* hv, const double* sx, const double* ss, double dw,
                    double dc, int mem) {
  if (!K || !hv || !sx || !ss) return GN_ERR_INVALID;
  if (is_full(mem) && !K->ctx) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  const double *dh = hv, *dsx = sx, *dss = ss;
  if (!is_device(mem)) {
    const int64_t n = is_full(mem) ? K->ctx->d.nh : K->nh;
    K->sh.upload(hv, n, K->stream);
    K->ssx.upload(sx, K->n, K->stream);
    K->sss.upload(ss, K->m, K->stream);
    dh = K->sh.p; dsx = K->ssx.p; dss = K->sss.p;
  }
  order_after_values(K, false, true);
  gnb::kkt_assemble(K, dh, dsx, dss, dw, dc, is_full(mem));
  if (!is_async(mem)) GN_CK(cudaStreamSynchronize(K->stream));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_set_jacobian_x(gn_kkt* K, const double* x, int mem) {
  if (!K || !x) return GN_ERR_INVALID;
  if (!gnb::opf_fused_ready(K)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(K->device);
  const double* dx = x;
  if (!is_device(mem)) {
    K->sj.upload(x, K->ctx->d.n, K->stream);
    dx = K->sj.p;
  }
  order_after_values(K, true, false);
  gnb::opf_set_jacobian_fused(K, dx);
  if (!is_async(mem)) GN_CK(cudaStreamSynchronize(K->stream));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_assemble_x(gn_kkt* K, const double* x, const double* w, double ow, const double* sx,
                      const double* ss, double dw, double dc, int mem) {
  if (!K || !x || !w || !sx || !ss) return GN_ERR_INVALID;
  if (!gnb::opf_fused_ready(K)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(K->device);
  const double *dx = x, *dwt = w, *dsx = sx, *dss = ss;
  if (!is_device(mem)) {
    K->sj.upload(x, K->ctx->d.n, K->stream);
    K->sh.upload(w, K->m, K->stream);
    K->ssx.upload(sx, K->n, K->stream);
    K->sss.upload(ss, K->m, K->stream);
    dx = K->sj.p; dwt = K->sh.p; dsx = K->ssx.p; dss = K->sss.p;
  }
  order_after_values(K, false, true);
  gnb::opf_assemble_fused(K, dx, dwt, ow, dsx, dss, dw, dc);
  if (!is_async(mem)) GN_CK(cudaStreamSynchronize(K->stream));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_update_x(gn_kkt* K, const double* x, const double* w, double ow, const double* sx,
                    const double* ss, double dw, double dc, int mem) {
  if (!K || !x || !w || !sx || !ss) return GN_ERR_INVALID;
  if (!gnb::opf_fused_ready(K)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(K->device);
  const double *dx = x, *dwt = w, *dsx = sx, *dss = ss;
  if (!is_device(mem)) {
    K->sj.upload(x, K->ctx->d.n, K->stream);
    K->sh.upload(w, K->m, K->stream);
    K->ssx.upload(sx, K->n, K->stream);
    K->sss.upload(ss, K->m, K->stream);
    dx = K->sj.p; dwt = K->sh.p; dsx = K->ssx.p; dss = K->sss.p;
  }
  order_after_values(K, true, true);
  gnb::opf_update_fused(K, dx, dwt, ow, dsx, dss, dw, dc);
  if (!is_async(mem)) GN_CK(cudaStreamSynchronize(K->stream));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_values(gn_kkt* K, double* av, double* mv, int mem) {
  if (!K) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  // device modes accept any UVA-addressable destination (device or pinned host memory)
  if (is_device(mem)) {
    if (av && K->annz)
      GN_CK(cudaMemcpyAsync(av, K->avals.p, sizeof(double) * K->annz, cudaMemcpyDefault, K->stream));
    if (mv && K->mnnz)
      GN_CK(cudaMemcpyAsync(mv, K->mvals.p, sizeof(double) * K->mnnz, cudaMemcpyDefault, K->stream));
  } else {
    if (av && K->annz) gnb::d2h(av, K->avals.p, sizeof(double) * K->annz, K->stream);
    if (mv && K->mnnz) gnb::d2h(mv, K->mvals.p, sizeof(double) * K->mnnz, K->stream);
  }
  if (!is_async(mem)) GN_CK(cudaStreamSynchronize(K->stream));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_values_start(gn_kkt* K, double* av, double* mv) {
  if (!K) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  if (!K->vstream) {
    GN_CK(cudaStreamCreateWithFlags(&K->vstream, cudaStreamNonBlocking));
    GN_CK(cudaEventCreateWithFlags(&K->vstart, cudaEventDisableTiming));
    GN_CK(cudaEventCreateWithFlags(&K->vdone, cudaEventDisableTiming));
  }
  GN_CK(cudaEventRecord(K->vstart, K->stream));
  GN_CK(cudaStreamWaitEvent(K->vstream, K->vstart, 0));
  if (av && K->annz)
    GN_CK(cudaMemcpyAsync(av, K->avals.p, sizeof(double) * K->annz, cudaMemcpyDefault, K->vstream));
  if (mv && K->mnnz)
    GN_CK(cudaMemcpyAsync(mv, K->mvals.p, sizeof(double) * K->mnnz, cudaMemcpyDefault, K->vstream));
  GN_CK(cudaEventRecord(K->vdone, K->vstream));
  K->vpend_a = K->vpend_a || (av && K->annz);
  K->vpend_m = K->vpend_m || (mv && K->mnnz);
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_values_wait(gn_kkt* K) {
  if (!K) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  if (K->vdone) GN_CK(cudaEventSynchronize(K->vdone));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_values_ptr(gn_kkt* K, const double** av, const double** mv) {
  if (!K) return GN_ERR_INVALID;
  if (av) *av = K->avals.p;
  if (mv) *mv = K->mvals.p;
  return GN_OK;
}

// ------------------------------------------------------------ test support
namespace {
__global__ void k_guard_fill(int64_t n, unsigned long long* p, unsigned long long v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
__global__ void k_guard_count(int64_t n, int64_t body, const unsigned long long* p,
                              unsigned long long v, unsigned long long* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i < body && p[i] == v) atomicAdd(out, 1ull);        // slot never written
  if (i >= body && p[i] != v) atomicAdd(out + 1, 1ull);   // guard band touched
}
}  // namespace

int gn_host_alloc(size_t bytes, void** out) {
  if (!out) return GN_ERR_INVALID;
  *out = nullptr;
  if (bytes == 0) return GN_OK;
  if (cudaHostAlloc(out, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return GN_ERR_CUDA;
  }
  return GN_OK;
}
int gn_host_free(void* p) {
  if (p && cudaFreeHost(p) != cudaSuccess) {
    cudaGetLastError();
    return GN_ERR_CUDA;
  }
  return GN_OK;
}

int gn_debug_kkt_guard(gn_kkt* K, int fill, uint64_t pattern, int64_t* out4) {
  if (!K || (!fill && !out4)) return GN_ERR_INVALID;
  API_TRY
  set_device(K->device);
  cudaStream_t s = K->stream;
  struct B { double* p; int64_t body; } bufs[2] = {{K->avals.p, K->annz}, {K->mvals.p, K->mnnz}};
  DBuf<unsigned long long> cnt;
  if (!fill) {
    cnt.alloc(4);
    GN_CK(cudaMemsetAsync(cnt.p, 0, 4 * sizeof(unsigned long long), s));
  }
  for (int b = 0; b < 2; ++b) {
    const int64_t n = bufs[b].body + gnb::kGuard;
    auto* p = reinterpret_cast<unsigned long long*>(bufs[b].p);
    const unsigned g = (unsigned)((n + 255) / 256);
    if (fill) k_guard_fill<<<g, 256, 0, s>>>(n, p, pattern);
    else k_guard_count<<<g, 256, 0, s>>>(n, bufs[b].body, p, pattern, cnt.p + 2 * b);
  }
  GN_CK(cudaGetLastError());
  if (!fill) {
    unsigned long long h[4];
    GN_CK(cudaMemcpyAsync(h, cnt.p, sizeof h, cudaMemcpyDeviceToHost, s));
    GN_CK(cudaStreamSynchronize(s));
    for (int i = 0; i < 4; ++i) out4[i] = static_cast<int64_t>(h[i]);
  }
  GN_CK(cudaStreamSynchronize(s));
  return GN_OK;
  API_CATCH(nullptr)
}

int gn_kkt_set_grid_cap(gn_kkt* K, int ctas_per_sm) {
  if (!K || ctas_per_sm < 0) return GN_ERR_INVALID;
  gnb::opf_set_grid_cap(K, ctas_per_sm);
  return GN_OK;
}

int gn_kkt_set_algorithm(gn_kkt* K, int algo) {
  if (!K || algo < 0 || algo > 2) return GN_ERR_INVALID;
  if (algo == 2 && !K->ctx) return GN_ERR_INVALID;
  K->algo = algo;
  return GN_OK;
}

int gn_compress_to_csc(int32_t nrows, int32_t ncols, int64_t nnz, const int32_t* rows,
                       const int32_t* cols, int32_t* colptr, int32_t* rowidx, int32_t* slot_map,
                       int32_t* nnz_out, gn_error* err) {
  if (nnz < 0 || nrows < 0 || ncols < 0) return fail(err, GN_ERR_INVALID, "negative size");
  API_TRY
  cudaStream_t s = nullptr;
  GN_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct Guard { cudaStream_t s; ~Guard() { cudaStreamDestroy(s); } } guard{s};
  for (int64_t k = 0; k < nnz; ++k)
    if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols)
      throw Error(GN_ERR_INVALID, "compress_to_csc: coordinate out of range");
  std::vector<uint64_t> key(static_cast<size_t>(nnz));
  for (int64_t k = 0; k < nnz; ++k) key[k] = (uint64_t)cols[k] * (uint64_t)nrows + (uint64_t)rows[k];
  DBuf<uint64_t> dk;
  dk.upload(key.data(), key.size(), s);
  gnb::Csc out;
  gnb::compress_keys(dk.p, nnz, nrows, ncols, out, s);
  if (colptr) GN_CK(cudaMemcpyAsync(colptr, out.ptr.p, sizeof(int32_t) * (ncols + 1), cudaMemcpyDeviceToHost, s));
  if (rowidx && out.nnz) GN_CK(cudaMemcpyAsync(rowidx, out.idx.p, sizeof(int32_t) * out.nnz, cudaMemcpyDeviceToHost, s));
  if (slot_map && nnz) GN_CK(cudaMemcpyAsync(slot_map, out.slot.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, s));
  GN_CK(cudaStreamSynchronize(s));
  if (nnz_out) *nnz_out = out.nnz;
  return ok(err);
  API_CATCH(err)
}

}  // extern "C"

// ------------------------------------------------- device-resident IPM vector ops
namespace {
int ipm_mode(int mem) { return is_device(mem) ? GN_OK : GN_ERR_UNSUPPORTED; }
int ipm_done(gn_ipm* P, int mem) {
  if (!is_async(mem)) GN_CK(cudaStreamSynchronize(P->K->stream));
  return GN_OK;
}
}  // namespace

extern "C" {

int gn_ipm_create(gn_kkt* K, const double* xl, const double* xu, const double* sl,
                  const double* su, int mem, gn_ipm** out, gn_error* err) {
  if (!K || !out) return fail(err, GN_ERR_INVALID, "null argument");
  if (!K->ctx) return fail(err, GN_ERR_INVALID, "gn_ipm_create needs a gn_kkt_create_lifted KKT");
  if ((K->n && (!xl || !xu)) || (K->m && (!sl || !su))) return fail(err, GN_ERR_INVALID, "null bounds");
  API_TRY
  set_device(K->device);
  *out = gnb::ipm_create(K, xl, xu, sl, su, is_device(mem));
  ++K->refs;
  return ok(err);
  API_CATCH(err)
}

int gn_ipm_destroy(gn_ipm* P) {
  if (!P) return GN_OK;
  cudaSetDevice(P->device);
  cudaStreamSynchronize(P->K->stream);
  gn_kkt* K = P->K;
  delete P;
  if (--K->refs == 0 && K->closed) kkt_free(K);
  return GN_OK;
}

int gn_ipm_jac_transpose_multiply(gn_ipm* P, const double* jv, const double* y, double* out,
                                  int mem) {
  if (!P || !jv || !y || !out) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_jac_t(P, jv, y, out, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_jac_multiply(gn_ipm* P, const double* jv, const double* x, double* out, int mem) {
  if (!P || !jv || !x || !out) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_jac(P, jv, x, out, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_residuals(gn_ipm* P, const gn_iterate* it, const double* grad, const double* g,
                     const double* jv, double mu, const gn_residuals* r, int mem) {
  if (!P || !it || !grad || !g || !jv || !r) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_residuals(P, *it, grad, g, jv, mu, *r, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_bound_condensation(gn_ipm* P, const gn_iterate* it, const gn_residuals* r,
                              double* sx, double* ss, double* qx, double* qs, int mem) {
  if (!P || !it || !r || !sx || !ss || !qx || !qs) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_condense(P, *it, *r, sx, ss, qx, qs, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_fraction_to_boundary(gn_ipm* P, const gn_iterate* it, const gn_direction* d,
                                double tau, double* out2, int mem) {
  if (!P || !it || !d || !out2) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_ftb(P, *it, *d, tau, out2, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_barrier_value(gn_ipm* P, double f, const double* x, const double* s, double mu,
                         double* out, int mem) {
  if (!P || !x || !s || !out) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_barrier(P, f, x, s, mu, out, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_barrier_slope(gn_ipm* P, const double* grad, const gn_iterate* it,
                         const gn_direction* d, double mu, double* out, int mem) {
  if (!P || !grad || !it || !d || !out) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_slope(P, grad, *it, *d, mu, out, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_constraint_violation(gn_ipm* P, const double* g, const double* s, double* out,
                                int mem) {
  if (!P || !g || !s || !out) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_violation(P, g, s, out, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_kkt_error(gn_ipm* P, const gn_iterate* it, const gn_residuals* r, double mu,
                     double* out3, int mem) {
  if (!P || !it || !r || !out3) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_kkt_error(P, *it, *r, mu, out3, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_ipm_recover_bound_steps(gn_ipm* P, const gn_iterate* it, const gn_residuals* r,
                               const gn_direction* d, int mem) {
  if (!P || !it || !r || !d) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::ipm_recover(P, *it, *r, *d, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_kkt_solve_rhs(gn_ipm* P, const double* qx, const double* qs, const double* qy,
                     const double* ss, double dw, double dc, double* rhs, int mem) {
  if (!P || !qx || !qs || !qy || !ss || !rhs) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::kkt_solve_rhs(P, qx, qs, qy, ss, dw, dc, rhs, P->scratch.p, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

int gn_kkt_solve_finish(gn_ipm* P, const double* dx, const double* qs, const double* qy,
                        const double* ss, double dw, double dc, double* ds, double* dy, int mem) {
  if (!P || !dx || !qs || !qy || !ss || !ds || !dy) return GN_ERR_INVALID;
  if (ipm_mode(mem)) return GN_ERR_UNSUPPORTED;
  API_TRY
  set_device(P->device);
  gnb::kkt_solve_finish(P, dx, qs, qy, ss, dw, dc, ds, dy, P->K->stream);
  return ipm_done(P, mem);
  API_CATCH(nullptr)
}

}  // extern "C"
