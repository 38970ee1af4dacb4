/* oracle/gn_oracle.c — TEST INFRASTRUCTURE ONLY (the CPU checker).
 *
 * Plain-C restatement of the reference hot path, operation-for-operation, so
 * its outputs are bit-identical to the compiled reference on the same inputs
 * (pinned in tests/test_oracle.py).  The product (paper_2405_14032_b200/) never
 * links or calls this file.
 *
 *   tape AD (Dual, forward, reverse)   model/tape.hpp:14-210
 *   expression DAG -> postorder tape   model/expr.hpp:37-86, tape.hpp:84-116
 *   the 12 OPF patterns + layout       power/opf.hpp:100-355
 *   freeze (J/H COO slot order)        model/pattern_model.hpp:158-207
 *   evaluate_*                         model/pattern_model.hpp:278-436
 *   lifted filter                      ipm/lifted.hpp:25-100
 *   compress_to_csc / csr, scatter     sparse/matrix.hpp:45-106
 *   CondensedKkt ctor / set_jacobian / assemble   ipm/condensed.hpp:29-135
 */
#define _GNU_SOURCE
#include "gn_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_INF (1.0 / 0.0)

/* ------------------------------------------------------------------ tape */
/* Op order mirrors expr.hpp:11-26. */
typedef enum {
  OP_CONST, OP_REAL, OP_VAR, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_NEG,
  OP_SIN, OP_COS, OP_SQRT, OP_LOG, OP_EXP, OP_POW
} op_t;

typedef struct node {
  op_t op;
  struct node *a, *b;
  double c;
  int field;
  int pos; /* tape position once emitted (dedupe by node identity, tape.hpp:95-96) */
} node;

#define POOL 64
typedef struct { node n[POOL]; int used; } pool_t;

static node* mk(pool_t* p, op_t op, node* a, node* b, double c, int field) {
  node* x = &p->n[p->used++];
  x->op = op; x->a = a; x->b = b; x->c = c; x->field = field; x->pos = -1;
  return x;
}
#define VAR(k) mk(P, OP_VAR, 0, 0, 0.0, (k))
#define REAL(k) mk(P, OP_REAL, 0, 0, 0.0, (k))
#define ADD(x, y) mk(P, OP_ADD, (x), (y), 0.0, -1)
#define SUB(x, y) mk(P, OP_SUB, (x), (y), 0.0, -1)
#define MUL(x, y) mk(P, OP_MUL, (x), (y), 0.0, -1)
#define NEG(x) mk(P, OP_NEG, (x), 0, 0.0, -1)
#define SIN(x) mk(P, OP_SIN, (x), 0, 0.0, -1)
#define COS(x) mk(P, OP_COS, (x), 0, 0.0, -1)
#define SQUARE(x) mk(P, OP_POW, (x), 0, 2.0, -1)

typedef struct { op_t op; int a, b, field; double c; } instr;
typedef struct { instr code[POOL]; int len; int nvar, nreal; } tape;

static int emit(const node* n0, tape* t) {
  node* n = (node*)n0;
  if (n->pos >= 0) return n->pos;
  instr in;
  in.op = n->op;
  in.a = n->a ? emit(n->a, t) : -1;
  in.b = n->b ? emit(n->b, t) : -1;
  in.field = n->field;
  in.c = n->c;
  if (n->op == OP_VAR && n->field + 1 > t->nvar) t->nvar = n->field + 1;
  if (n->op == OP_REAL && n->field + 1 > t->nreal) t->nreal = n->field + 1;
  t->code[t->len] = in;
  n->pos = t->len++;
  return n->pos;
}

static void compile(node* root, tape* t) {
  memset(t, 0, sizeof *t);
  emit(root, t);
}

/* Dual number (tape.hpp:14-47). */
typedef struct { double v, d; } dual;
static inline dual D1(double v) { dual r = {v, 0.0}; return r; }
static inline dual D2(double v, double d) { dual r = {v, d}; return r; }
static inline dual dadd(dual a, dual b) { return D2(a.v + b.v, a.d + b.d); }
static inline dual dsub(dual a, dual b) { return D2(a.v - b.v, a.d - b.d); }
static inline dual dneg(dual a) { return D2(-a.v, -a.d); }
static inline dual dmul(dual a, dual b) { return D2(a.v * b.v, a.d * b.v + a.v * b.d); }
static inline dual ddiv(dual a, dual b) {
  const double q = a.v / b.v;
  return D2(q, (a.d - q * b.d) / b.v);
}
static inline dual dsin(dual a) { return D2(sin(a.v), cos(a.v) * a.d); }
static inline dual dcos(dual a) { return D2(cos(a.v), -sin(a.v) * a.d); }
static inline dual dsqrt(dual a) {
  const double s = sqrt(a.v);
  return D2(s, 0.5 * a.d / s);
}
static inline dual dlog(dual a) { return D2(log(a.v), a.d / a.v); }
static inline dual dexp(dual a) {
  const double e = exp(a.v);
  return D2(e, e * a.d);
}
static inline dual dpow(dual a, double c) { return D2(pow(a.v, c), c * pow(a.v, c - 1.0) * a.d); }

static int pow_domain_ok(double u, double c) { /* tape.hpp:119-123 */
  const int integral = (c == nearbyint(c));
  if (integral) return c >= 0.0 || u != 0.0;
  return u > 0.0;
}

/* tape_forward<double> (tape.hpp:127-163) */
static int fwd_d(const tape* t, const double* reals, const double* x, double* v) {
  for (int i = 0; i < t->len; ++i) {
    const instr* in = &t->code[i];
    switch (in->op) {
      case OP_CONST: v[i] = in->c; break;
      case OP_REAL: v[i] = reals[in->field]; break;
      case OP_VAR: v[i] = x[in->field]; break;
      case OP_ADD: v[i] = v[in->a] + v[in->b]; break;
      case OP_SUB: v[i] = v[in->a] - v[in->b]; break;
      case OP_MUL: v[i] = v[in->a] * v[in->b]; break;
      case OP_DIV:
        if (v[in->b] == 0.0) return 0;
        v[i] = v[in->a] / v[in->b];
        break;
      case OP_NEG: v[i] = -v[in->a]; break;
      case OP_SIN: v[i] = sin(v[in->a]); break;
      case OP_COS: v[i] = cos(v[in->a]); break;
      case OP_SQRT:
        if (!(v[in->a] > 0.0)) return 0;
        v[i] = sqrt(v[in->a]);
        break;
      case OP_LOG:
        if (!(v[in->a] > 0.0)) return 0;
        v[i] = log(v[in->a]);
        break;
      case OP_EXP: v[i] = exp(v[in->a]); break;
      case OP_POW:
        if (!pow_domain_ok(v[in->a], in->c)) return 0;
        v[i] = pow(v[in->a], in->c);
        break;
    }
  }
  return 1;
}

/* tape_forward<Dual> */
static int fwd_dual(const tape* t, const double* reals, const dual* x, dual* v) {
  for (int i = 0; i < t->len; ++i) {
    const instr* in = &t->code[i];
    switch (in->op) {
      case OP_CONST: v[i] = D1(in->c); break;
      case OP_REAL: v[i] = D1(reals[in->field]); break;
      case OP_VAR: v[i] = x[in->field]; break;
      case OP_ADD: v[i] = dadd(v[in->a], v[in->b]); break;
      case OP_SUB: v[i] = dsub(v[in->a], v[in->b]); break;
      case OP_MUL: v[i] = dmul(v[in->a], v[in->b]); break;
      case OP_DIV:
        if (v[in->b].v == 0.0) return 0;
        v[i] = ddiv(v[in->a], v[in->b]);
        break;
      case OP_NEG: v[i] = dneg(v[in->a]); break;
      case OP_SIN: v[i] = dsin(v[in->a]); break;
      case OP_COS: v[i] = dcos(v[in->a]); break;
      case OP_SQRT:
        if (!(v[in->a].v > 0.0)) return 0;
        v[i] = dsqrt(v[in->a]);
        break;
      case OP_LOG:
        if (!(v[in->a].v > 0.0)) return 0;
        v[i] = dlog(v[in->a]);
        break;
      case OP_EXP: v[i] = dexp(v[in->a]); break;
      case OP_POW:
        if (!pow_domain_ok(v[in->a].v, in->c)) return 0;
        v[i] = dpow(v[in->a], in->c);
        break;
    }
  }
  return 1;
}

/* tape_reverse<double> (tape.hpp:168-210) */
static void rev_d(const tape* t, const double* v, double* adj, double seed, double* xbar) {
  const int len = t->len;
  for (int i = 0; i < len; ++i) adj[i] = 0.0;
  adj[len - 1] = seed;
  for (int i = len - 1; i >= 0; --i) {
    const double a = adj[i];
    if (a == 0.0) continue;
    const instr* in = &t->code[i];
    switch (in->op) {
      case OP_CONST: case OP_REAL: break;
      case OP_VAR: xbar[in->field] += a; break;
      case OP_ADD: adj[in->a] += a; adj[in->b] += a; break;
      case OP_SUB: adj[in->a] += a; adj[in->b] -= a; break;
      case OP_MUL:
        adj[in->a] += a * v[in->b];
        adj[in->b] += a * v[in->a];
        break;
      case OP_DIV:
        adj[in->a] += a / v[in->b];
        adj[in->b] -= a * v[i] / v[in->b];
        break;
      case OP_NEG: adj[in->a] -= a; break;
      case OP_SIN: adj[in->a] += a * cos(v[in->a]); break;
      case OP_COS: adj[in->a] -= a * sin(v[in->a]); break;
      case OP_SQRT: adj[in->a] += a * 0.5 / v[i]; break;
      case OP_LOG: adj[in->a] += a / v[in->a]; break;
      case OP_EXP: adj[in->a] += a * v[i]; break;
      case OP_POW: adj[in->a] += a * in->c * pow(v[in->a], in->c - 1.0); break;
    }
  }
}

/* tape_reverse<Dual> */
static void rev_dual(const tape* t, const dual* v, dual* adj, dual seed, dual* xbar) {
  const int len = t->len;
  for (int i = 0; i < len; ++i) adj[i] = D1(0.0);
  adj[len - 1] = seed;
  for (int i = len - 1; i >= 0; --i) {
    const dual a = adj[i];
    if (a.v == 0.0 && a.d == 0.0) continue;
    const instr* in = &t->code[i];
    switch (in->op) {
      case OP_CONST: case OP_REAL: break;
      case OP_VAR: xbar[in->field] = dadd(xbar[in->field], a); break;
      case OP_ADD:
        adj[in->a] = dadd(adj[in->a], a);
        adj[in->b] = dadd(adj[in->b], a);
        break;
      case OP_SUB:
        adj[in->a] = dadd(adj[in->a], a);
        adj[in->b] = dsub(adj[in->b], a);
        break;
      case OP_MUL:
        adj[in->a] = dadd(adj[in->a], dmul(a, v[in->b]));
        adj[in->b] = dadd(adj[in->b], dmul(a, v[in->a]));
        break;
      case OP_DIV:
        adj[in->a] = dadd(adj[in->a], ddiv(a, v[in->b]));
        adj[in->b] = dsub(adj[in->b], ddiv(dmul(a, v[i]), v[in->b]));
        break;
      case OP_NEG: adj[in->a] = dsub(adj[in->a], a); break;
      case OP_SIN: adj[in->a] = dadd(adj[in->a], dmul(a, dcos(v[in->a]))); break;
      case OP_COS: adj[in->a] = dsub(adj[in->a], dmul(a, dsin(v[in->a]))); break;
      case OP_SQRT: adj[in->a] = dadd(adj[in->a], ddiv(dmul(a, D1(0.5)), v[i])); break;
      case OP_LOG: adj[in->a] = dadd(adj[in->a], ddiv(a, v[in->a])); break;
      case OP_EXP: adj[in->a] = dadd(adj[in->a], dmul(a, v[i])); break;
      case OP_POW:
        adj[in->a] = dadd(adj[in->a], dmul(dmul(a, D1(in->c)), dpow(v[in->a], in->c - 1.0)));
        break;
    }
  }
}

/* ---------------------------------------------------------------- patterns */
/* The 12 expressions exactly as power/opf.hpp writes them (C++ operator
 * precedence made explicit).  Every var()/real() call is a fresh node; `dth`
 * is one shared node per expression (opf.hpp:309). */
enum {
  PT_COST, PT_BAL_P_FLOW, PT_BAL_Q_FLOW, PT_BAL_P_INJ, PT_BAL_Q_INJ, PT_BAL_P_LOAD,
  PT_BAL_Q_LOAD, PT_FLOW_P, PT_FLOW_Q, PT_THERMAL, PT_ANGLE, PT_RAMP, PT_KINDS
};

static void build_tape(int kind, tape* t) {
  pool_t pool;
  pool_t* P = &pool;
  pool.used = 0;
  node* e = 0;
  switch (kind) {
    case PT_COST: /* opf.hpp:245 real(0)*square(var(0)) + real(1)*var(0) + real(2) */
      e = ADD(ADD(MUL(REAL(0), SQUARE(VAR(0))), MUL(REAL(1), VAR(0))), REAL(2));
      break;
    case PT_BAL_P_FLOW: case PT_BAL_Q_FLOW: /* opf.hpp:260 real(0)*var(0) */
      e = MUL(REAL(0), VAR(0));
      break;
    case PT_BAL_P_INJ: case PT_BAL_Q_INJ: /* opf.hpp:275 var(0) */
      e = VAR(0);
      break;
    case PT_BAL_P_LOAD: case PT_BAL_Q_LOAD: /* opf.hpp:289 -real(0) */
      e = NEG(REAL(0));
      break;
    case PT_FLOW_P: { /* opf.hpp:310-314 */
      node* dth = SUB(VAR(3), VAR(4));
      e = SUB(VAR(0), SUB(MUL(REAL(0), SQUARE(VAR(1))),
                          MUL(MUL(VAR(1), VAR(2)),
                              ADD(MUL(REAL(0), COS(dth)), MUL(REAL(1), SIN(dth))))));
      break;
    }
    case PT_FLOW_Q: { /* opf.hpp:315-319 */
      node* dth = SUB(VAR(3), VAR(4));
      e = SUB(VAR(0), SUB(MUL(NEG(REAL(1)), SQUARE(VAR(1))),
                          MUL(MUL(VAR(1), VAR(2)),
                              SUB(MUL(REAL(0), SIN(dth)), MUL(REAL(1), COS(dth))))));
      break;
    }
    case PT_THERMAL: /* opf.hpp:331 square(var(0)) + square(var(1)) */
      e = ADD(SQUARE(VAR(0)), SQUARE(VAR(1)));
      break;
    case PT_ANGLE: case PT_RAMP: /* opf.hpp:340,350 var(0) - var(1) */
      e = SUB(VAR(0), VAR(1));
      break;
  }
  compile(e, t);
}

/* ------------------------------------------------------------------ model */
typedef struct {
  int kind;         /* PT_* */
  int is_objective;
  tape tp;
  int32_t nrec, k, nr;
  int32_t* vars;    /* nrec x k */
  double* reals;    /* nrec x nr */
  int32_t* rows;    /* nrec (flat rows) */
  int64_t jac_off, hess_off;
  int32_t* dbl;     /* double_slots */
  int64_t ndbl;
} pattern;

typedef struct {
  int32_t n_free;
  int32_t *free_of_full, *full_of_free;
  int64_t nj, nh;
  int32_t *jr, *jc, *jpick, *hr, *hc, *hpick;
  double *sl, *su;
} lifted_t;

struct or_model {
  int32_t T, N, L, G, D, LT, GR;
  int32_t n, m;
  double *xl, *xu, *xs, *rl, *ru;
  pattern pat[PT_KINDS];
  int npat;
  int64_t nj, nh;
  int32_t *jr, *jc, *hr, *hc;
  double* contrib;
  int has_lifted;
  lifted_t lift;
};

typedef struct { int32_t *vars, *rows; double* reals; int32_t n, cap, k, nr; } recs;

static void rec_init(recs* r, int k, int nr, int cap) {
  r->k = k; r->nr = nr; r->n = 0; r->cap = cap > 0 ? cap : 1;
  r->vars = (int32_t*)malloc(sizeof(int32_t) * (size_t)r->cap * (k > 0 ? k : 1));
  r->reals = (double*)malloc(sizeof(double) * (size_t)r->cap * (nr > 0 ? nr : 1));
  r->rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)r->cap);
}
static void rec_add(recs* r, const int32_t* v, const double* re, int32_t row) {
  for (int i = 0; i < r->k; ++i) r->vars[(size_t)r->n * r->k + i] = v[i];
  for (int i = 0; i < r->nr; ++i) r->reals[(size_t)r->n * r->nr + i] = re[i];
  r->rows[r->n] = row;
  r->n++;
}

static void add_pattern(or_model* m, int kind, int is_obj, recs* r) {
  pattern* p = &m->pat[m->npat++];
  memset(p, 0, sizeof *p);
  p->kind = kind;
  p->is_objective = is_obj;
  build_tape(kind, &p->tp);
  p->nrec = r->n; p->k = r->k; p->nr = r->nr;
  p->vars = r->vars; p->reals = r->reals; p->rows = r->rows;
}

static double* spread(int32_t count, int32_t T, const double* per, double fill, int use_fill) {
  double* o = (double*)malloc(sizeof(double) * ((size_t)count * T + 1));
  for (int32_t e = 0; e < count; ++e)
    for (int32_t t = 0; t < T; ++t) o[(size_t)e * T + t] = use_fill ? fill : per[e];
  return o;
}

or_model* or_model_create(const or_network* net, int32_t T, const double* scale, char* err,
                          int errlen) {
  const int32_t N = net->n_bus, L = net->n_line, G = net->n_gen, D = net->n_load;
  if (net->reference_bus < 0 || net->reference_bus >= N) {
    if (err) snprintf(err, (size_t)errlen, "opf: network has no reference bus");
    return 0;
  }
  if (T < 1) {
    if (err) snprintf(err, (size_t)errlen, "load profile: need at least one period");
    return 0;
  }
  or_model* m = (or_model*)calloc(1, sizeof(or_model));
  m->T = T; m->N = N; m->L = L; m->G = G; m->D = D;
  /* thermal lines / ramp gens (opf.hpp:116-122) */
  int32_t* thermal = (int32_t*)malloc(sizeof(int32_t) * (L + 1));
  int32_t* rampg = (int32_t*)malloc(sizeof(int32_t) * (G + 1));
  int32_t LT = 0, GR = 0;
  for (int32_t l = 0; l < L; ++l)
    if (net->line_smax[l] < OR_INF) thermal[LT++] = l;
  if (T >= 2)
    for (int32_t g = 0; g < G; ++g)
      if (net->gen_ramp[g] < OR_INF) rampg[GR++] = g;
  m->LT = LT; m->GR = GR;

  /* variable blocks pg, qg, p, q, v, th (opf.hpp:135-183) */
  const int32_t pg0 = 0, qg0 = G * T, p0 = 2 * G * T, q0 = p0 + L * T, v0 = q0 + L * T,
                th0 = v0 + N * T;
  m->n = th0 + N * T;
  m->xl = (double*)malloc(sizeof(double) * ((size_t)m->n + 1));
  m->xu = (double*)malloc(sizeof(double) * ((size_t)m->n + 1));
  m->xs = (double*)malloc(sizeof(double) * ((size_t)m->n + 1));
#define PUT(dst, off, cnt, src) memcpy((dst) + (off), (src), sizeof(double) * (size_t)(cnt) * T)
  {
    double* a;
    a = spread(G, T, net->gen_pmin, 0, 0); PUT(m->xl, pg0, G, a); free(a);
    a = spread(G, T, net->gen_pmax, 0, 0); PUT(m->xu, pg0, G, a); free(a);
    a = spread(G, T, net->gen_pstart, 0, 0); PUT(m->xs, pg0, G, a); free(a);
    a = spread(G, T, net->gen_qmin, 0, 0); PUT(m->xl, qg0, G, a); free(a);
    a = spread(G, T, net->gen_qmax, 0, 0); PUT(m->xu, qg0, G, a); free(a);
    a = spread(G, T, net->gen_qstart, 0, 0); PUT(m->xs, qg0, G, a); free(a);
    double* ps = (double*)malloc(sizeof(double) * (L + 1));
    double* qs = (double*)malloc(sizeof(double) * (L + 1));
    for (int32_t l = 0; l < L; ++l) { /* line_flow, network.hpp:76-82 */
      const double vm = net->vm_start[net->line_from[l]], vn = net->vm_start[net->line_to[l]];
      const double dth = net->va_start[net->line_from[l]] - net->va_start[net->line_to[l]];
      const double c = cos(dth), s = sin(dth), g = net->line_g[l], b = net->line_b[l];
      ps[l] = g * vm * vm - vm * vn * (g * c + b * s);
      qs[l] = -b * vm * vm - vm * vn * (g * s - b * c);
    }
    a = spread(L, T, 0, -OR_INF, 1); PUT(m->xl, p0, L, a); PUT(m->xl, q0, L, a); free(a);
    a = spread(L, T, 0, OR_INF, 1); PUT(m->xu, p0, L, a); PUT(m->xu, q0, L, a); free(a);
    a = spread(L, T, ps, 0, 0); PUT(m->xs, p0, L, a); free(a);
    a = spread(L, T, qs, 0, 0); PUT(m->xs, q0, L, a); free(a);
    free(ps); free(qs);
    a = spread(N, T, net->bus_vmin, 0, 0); PUT(m->xl, v0, N, a); free(a);
    a = spread(N, T, net->bus_vmax, 0, 0); PUT(m->xu, v0, N, a); free(a);
    a = spread(N, T, net->vm_start, 0, 0); PUT(m->xs, v0, N, a); free(a);
    const int32_t ref = net->reference_bus;
    for (int32_t n = 0; n < N; ++n)
      for (int32_t t = 0; t < T; ++t) {
        const size_t i = (size_t)th0 + (size_t)n * T + t;
        m->xl[i] = n == ref ? 0.0 : -OR_INF;
        m->xu[i] = n == ref ? 0.0 : OR_INF;
        m->xs[i] = n == ref ? 0.0 : net->va_start[n];
      }
  }
#undef PUT
  /* row blocks (opf.hpp:186-230) */
  const int32_t bal_p0 = 0, bal_q0 = N * T, flow_p0 = 2 * N * T, flow_q0 = flow_p0 + L * T,
                therm0 = flow_q0 + L * T, ang0 = therm0 + LT * T, ramp0 = ang0 + L * T;
  const int32_t ramp_rows = GR * (T - 1 > 0 ? T - 1 : 0);
  m->m = ramp0 + ramp_rows;
  m->rl = (double*)malloc(sizeof(double) * ((size_t)m->m + 1));
  m->ru = (double*)malloc(sizeof(double) * ((size_t)m->m + 1));
  for (int32_t i = 0; i < therm0; ++i) m->rl[i] = m->ru[i] = 0.0;
  for (int32_t k = 0; k < LT; ++k) {
    const double s = net->line_smax[thermal[k]];
    for (int32_t t = 0; t < T; ++t) {
      m->rl[therm0 + k * T + t] = -OR_INF;
      m->ru[therm0 + k * T + t] = s * s;
    }
  }
  for (int32_t l = 0; l < L; ++l)
    for (int32_t t = 0; t < T; ++t) {
      m->rl[ang0 + l * T + t] = net->line_amin[l];
      m->ru[ang0 + l * T + t] = net->line_amax[l];
    }
  for (int32_t k = 0; k < GR; ++k) {
    const double r = net->gen_ramp[rampg[k]];
    for (int32_t s = 0; s < T - 1; ++s) {
      m->rl[ramp0 + k * (T - 1) + s] = -r;
      m->ru[ramp0 + k * (T - 1) + s] = r;
    }
  }

  /* patterns in registration order (opf.hpp:236-351); rows stored flat */
  recs r, r2;
  int32_t v[5];
  double re[3];
  rec_init(&r, 1, 3, G * T);
  for (int32_t g = 0; g < G; ++g)
    for (int32_t t = 0; t < T; ++t) {
      v[0] = pg0 + g * T + t;
      re[0] = net->gen_c2[g]; re[1] = net->gen_c1[g]; re[2] = net->gen_c0[g];
      rec_add(&r, v, re, -1);
    }
  add_pattern(m, PT_COST, 1, &r);

  rec_init(&r, 1, 1, 2 * L * T);
  rec_init(&r2, 1, 1, 2 * L * T);
  for (int32_t l = 0; l < L; ++l)
    for (int32_t t = 0; t < T; ++t) {
      const int32_t fr = net->line_from[l], to = net->line_to[l];
      v[0] = p0 + l * T + t; re[0] = 1.0; rec_add(&r, v, re, bal_p0 + to * T + t);
      re[0] = -1.0; rec_add(&r, v, re, bal_p0 + fr * T + t);
      v[0] = q0 + l * T + t; re[0] = 1.0; rec_add(&r2, v, re, bal_q0 + to * T + t);
      re[0] = -1.0; rec_add(&r2, v, re, bal_q0 + fr * T + t);
    }
  add_pattern(m, PT_BAL_P_FLOW, 0, &r);
  add_pattern(m, PT_BAL_Q_FLOW, 0, &r2);

  rec_init(&r, 1, 0, G * T);
  rec_init(&r2, 1, 0, G * T);
  for (int32_t g = 0; g < G; ++g)
    for (int32_t t = 0; t < T; ++t) {
      const int32_t bus = net->gen_bus[g];
      v[0] = pg0 + g * T + t; rec_add(&r, v, re, bal_p0 + bus * T + t);
      v[0] = qg0 + g * T + t; rec_add(&r2, v, re, bal_q0 + bus * T + t);
    }
  add_pattern(m, PT_BAL_P_INJ, 0, &r);
  add_pattern(m, PT_BAL_Q_INJ, 0, &r2);

  rec_init(&r, 0, 1, D * T);
  rec_init(&r2, 0, 1, D * T);
  for (int32_t j = 0; j < D; ++j)
    for (int32_t t = 0; t < T; ++t) {
      const int32_t bus = net->load_bus[j];
      /* MultiPeriodCase::pd/qd (network.hpp:166-171) */
      re[0] = net->load_p[j] * scale[(size_t)t * D + j];
      rec_add(&r, v, re, bal_p0 + bus * T + t);
      re[0] = net->load_q[j] * scale[(size_t)t * D + j];
      rec_add(&r2, v, re, bal_q0 + bus * T + t);
    }
  add_pattern(m, PT_BAL_P_LOAD, 0, &r);
  add_pattern(m, PT_BAL_Q_LOAD, 0, &r2);

  rec_init(&r, 5, 2, L * T);
  rec_init(&r2, 5, 2, L * T);
  for (int32_t l = 0; l < L; ++l)
    for (int32_t t = 0; t < T; ++t) {
      const int32_t fr = net->line_from[l], to = net->line_to[l];
      v[1] = v0 + fr * T + t; v[2] = v0 + to * T + t;
      v[3] = th0 + fr * T + t; v[4] = th0 + to * T + t;
      re[0] = net->line_g[l]; re[1] = net->line_b[l];
      v[0] = p0 + l * T + t; rec_add(&r, v, re, flow_p0 + l * T + t);
      v[0] = q0 + l * T + t; rec_add(&r2, v, re, flow_q0 + l * T + t);
    }
  add_pattern(m, PT_FLOW_P, 0, &r);
  add_pattern(m, PT_FLOW_Q, 0, &r2);

  if (LT > 0) {
    rec_init(&r, 2, 0, LT * T);
    for (int32_t k = 0; k < LT; ++k)
      for (int32_t t = 0; t < T; ++t) {
        const int32_t l = thermal[k];
        v[0] = p0 + l * T + t; v[1] = q0 + l * T + t;
        rec_add(&r, v, re, therm0 + k * T + t);
      }
    add_pattern(m, PT_THERMAL, 0, &r);
  }
  rec_init(&r, 2, 0, L * T);
  for (int32_t l = 0; l < L; ++l)
    for (int32_t t = 0; t < T; ++t) {
      v[0] = th0 + net->line_from[l] * T + t;
      v[1] = th0 + net->line_to[l] * T + t;
      rec_add(&r, v, re, ang0 + l * T + t);
    }
  add_pattern(m, PT_ANGLE, 0, &r);
  if (ramp_rows > 0) {
    rec_init(&r, 2, 0, ramp_rows);
    for (int32_t k = 0; k < GR; ++k)
      for (int32_t t = 1; t < T; ++t) {
        const int32_t g = rampg[k];
        v[0] = pg0 + g * T + t; v[1] = pg0 + g * T + t - 1;
        rec_add(&r, v, re, ramp0 + k * (T - 1) + (t - 1));
      }
    add_pattern(m, PT_RAMP, 0, &r);
  }
  free(thermal);
  free(rampg);

  /* freeze (pattern_model.hpp:158-207) */
  int64_t nj = 0, nh = 0;
  for (int i = 0; i < m->npat; ++i) {
    pattern* p = &m->pat[i];
    if (!p->is_objective) nj += (int64_t)p->nrec * p->k;
    nh += (int64_t)p->nrec * p->k * (p->k + 1) / 2;
  }
  m->jr = (int32_t*)malloc(sizeof(int32_t) * (nj + 1));
  m->jc = (int32_t*)malloc(sizeof(int32_t) * (nj + 1));
  m->hr = (int32_t*)malloc(sizeof(int32_t) * (nh + 1));
  m->hc = (int32_t*)malloc(sizeof(int32_t) * (nh + 1));
  nj = nh = 0;
  int32_t maxrec = 1;
  for (int i = 0; i < m->npat; ++i) {
    pattern* p = &m->pat[i];
    if (p->nrec > maxrec) maxrec = p->nrec;
    p->jac_off = -1;
    if (!p->is_objective) {
      p->jac_off = nj;
      for (int32_t q = 0; q < p->nrec; ++q)
        for (int32_t f = 0; f < p->k; ++f) {
          m->jr[nj] = p->rows[q];
          m->jc[nj] = p->vars[(size_t)q * p->k + f];
          ++nj;
        }
    }
    p->hess_off = nh;
    p->dbl = (int32_t*)malloc(sizeof(int32_t) * 16);
    int64_t cap = 16;
    for (int32_t q = 0; q < p->nrec; ++q) {
      const int32_t* vv = p->vars + (size_t)q * p->k;
      for (int32_t j = 0; j < p->k; ++j)
        for (int32_t ii = j; ii < p->k; ++ii) {
          const int32_t gi = vv[ii], gj = vv[j];
          m->hr[nh] = gi > gj ? gi : gj;
          m->hc[nh] = gi < gj ? gi : gj;
          if (ii != j && gi == gj) {
            if (p->ndbl == cap) {
              cap *= 2;
              p->dbl = (int32_t*)realloc(p->dbl, sizeof(int32_t) * cap);
            }
            p->dbl[p->ndbl++] = (int32_t)nh;
          }
          ++nh;
        }
    }
  }
  m->nj = nj;
  m->nh = nh;
  m->contrib = (double*)malloc(sizeof(double) * ((size_t)maxrec * 5 + 1));
  return m;
}

void or_model_free(or_model* m) {
  if (!m) return;
  for (int i = 0; i < m->npat; ++i) {
    free(m->pat[i].vars); free(m->pat[i].reals); free(m->pat[i].rows); free(m->pat[i].dbl);
  }
  free(m->xl); free(m->xu); free(m->xs); free(m->rl); free(m->ru);
  free(m->jr); free(m->jc); free(m->hr); free(m->hc); free(m->contrib);
  if (m->has_lifted) {
    lifted_t* L = &m->lift;
    free(L->free_of_full); free(L->full_of_free); free(L->jr); free(L->jc); free(L->jpick);
    free(L->hr); free(L->hc); free(L->hpick); free(L->sl); free(L->su);
  }
  free(m);
}

void or_model_sizes(const or_model* m, int64_t* s) {
  s[0] = m->n; s[1] = m->m; s[2] = m->nj; s[3] = m->nh; s[4] = m->LT; s[5] = m->GR;
}

void or_model_bounds(const or_model* m, double* xl, double* xu, double* xs, double* rl,
                     double* ru) {
  memcpy(xl, m->xl, sizeof(double) * m->n);
  memcpy(xu, m->xu, sizeof(double) * m->n);
  memcpy(xs, m->xs, sizeof(double) * m->n);
  memcpy(rl, m->rl, sizeof(double) * m->m);
  memcpy(ru, m->ru, sizeof(double) * m->m);
}

void or_model_structure(const or_model* m, int32_t* jr, int32_t* jc, int32_t* hr,
                        int32_t* hc) {
  memcpy(jr, m->jr, sizeof(int32_t) * m->nj);
  memcpy(jc, m->jc, sizeof(int32_t) * m->nj);
  memcpy(hr, m->hr, sizeof(int32_t) * m->nh);
  memcpy(hc, m->hc, sizeof(int32_t) * m->nh);
}


void or_model_offsets(const or_model* m, int64_t* jac_off, int64_t* hess_off,
                      int64_t* records) {
  for (int i = 0; i < 12; ++i) { jac_off[i] = -1; hess_off[i] = -1; records[i] = 0; }
  for (int i = 0; i < m->npat; ++i) {
    jac_off[i] = m->pat[i].jac_off;
    hess_off[i] = m->pat[i].hess_off;
    records[i] = m->pat[i].nrec;
  }
}

/* ------------------------------------------------------------- evaluation */
#define TAPE_MAX POOL
static void gather(const pattern* p, int32_t r, const double* x, double* xl) {
  const int32_t* vv = p->vars + (size_t)r * p->k;
  for (int32_t f = 0; f < p->k; ++f) xl[f] = x[vv[f]];
}
static const double* rec_reals(const pattern* p, int32_t r) {
  return p->reals + (size_t)r * p->nr;
}
static void set_fail(int32_t* fail, int pid, int32_t r) {
  if (fail) { fail[0] = pid; fail[1] = r; }
}

/* pattern_model.hpp:278-300 */
int or_eval_f(or_model* m, const double* x, double* out, int32_t* fail) {
  double vals[TAPE_MAX], xl[8];
  *out = 0.0;
  double total = 0.0;
  for (int pid = 0; pid < m->npat; ++pid) {
    const pattern* p = &m->pat[pid];
    if (!p->is_objective) continue;
    for (int32_t r = 0; r < p->nrec; ++r) {
      gather(p, r, x, xl);
      if (!fwd_d(&p->tp, rec_reals(p, r), xl, vals)) { set_fail(fail, pid, r); return 0; }
      const double v = vals[p->tp.len - 1];
      if (!isfinite(v)) { set_fail(fail, pid, r); return 0; }
      m->contrib[r] = v;
    }
    for (int32_t r = 0; r < p->nrec; ++r) total += m->contrib[r];
  }
  *out = total;
  return 1;
}

/* pattern_model.hpp:302-326 */
int or_eval_g(or_model* m, const double* x, double* g, int32_t* fail) {
  double vals[TAPE_MAX], xl[8];
  for (int32_t i = 0; i < m->m; ++i) g[i] = 0.0;
  for (int pid = 0; pid < m->npat; ++pid) {
    const pattern* p = &m->pat[pid];
    if (p->is_objective) continue;
    for (int32_t r = 0; r < p->nrec; ++r) {
      gather(p, r, x, xl);
      if (!fwd_d(&p->tp, rec_reals(p, r), xl, vals)) { set_fail(fail, pid, r); return 0; }
      const double v = vals[p->tp.len - 1];
      if (!isfinite(v)) { set_fail(fail, pid, r); return 0; }
      m->contrib[r] = v;
    }
    for (int32_t r = 0; r < p->nrec; ++r) g[p->rows[r]] += m->contrib[r];
  }
  return 1;
}

/* pattern_model.hpp:328-359 */
int or_eval_grad(or_model* m, const double* x, double* grad, int32_t* fail) {
  double vals[TAPE_MAX], adj[TAPE_MAX], xl[8], xbar[8];
  for (int32_t i = 0; i < m->n; ++i) grad[i] = 0.0;
  for (int pid = 0; pid < m->npat; ++pid) {
    const pattern* p = &m->pat[pid];
    if (!p->is_objective) continue;
    const int32_t k = p->k;
    for (int32_t r = 0; r < p->nrec; ++r) {
      gather(p, r, x, xl);
      if (!fwd_d(&p->tp, rec_reals(p, r), xl, vals)) { set_fail(fail, pid, r); return 0; }
      for (int32_t f = 0; f < k; ++f) xbar[f] = 0.0;
      rev_d(&p->tp, vals, adj, 1.0, xbar);
      for (int32_t f = 0; f < k; ++f) {
        if (!isfinite(xbar[f])) { set_fail(fail, pid, r); return 0; }
        m->contrib[(size_t)r * k + f] = xbar[f];
      }
    }
    for (int32_t r = 0; r < p->nrec; ++r) {
      const int32_t* vv = p->vars + (size_t)r * k;
      for (int32_t f = 0; f < k; ++f) grad[vv[f]] += m->contrib[(size_t)r * k + f];
    }
  }
  return 1;
}

/* pattern_model.hpp:361-388 */
int or_eval_jac(or_model* m, const double* x, double* out, int32_t* fail) {
  double vals[TAPE_MAX], adj[TAPE_MAX], xl[8], xbar[8];
  for (int pid = 0; pid < m->npat; ++pid) {
    const pattern* p = &m->pat[pid];
    if (p->is_objective) continue;
    const int32_t k = p->k;
    for (int32_t r = 0; r < p->nrec; ++r) {
      gather(p, r, x, xl);
      if (!fwd_d(&p->tp, rec_reals(p, r), xl, vals)) { set_fail(fail, pid, r); return 0; }
      for (int32_t f = 0; f < k; ++f) xbar[f] = 0.0;
      rev_d(&p->tp, vals, adj, 1.0, xbar);
      double* o = out + p->jac_off + (size_t)r * k;
      for (int32_t f = 0; f < k; ++f) {
        if (!isfinite(xbar[f])) { set_fail(fail, pid, r); return 0; }
        o[f] = xbar[f];
      }
    }
  }
  return 1;
}

/* pattern_model.hpp:393-436 (forward-over-reverse, one dual sweep per field) */
int or_eval_hess(or_model* m, const double* x, const double* w, double ow, double* out,
                 int32_t* fail) {
  dual vals[TAPE_MAX], adj[TAPE_MAX], xd[8], xbar[8];
  double xl[8];
  for (int pid = 0; pid < m->npat; ++pid) {
    const pattern* p = &m->pat[pid];
    const int32_t k = p->k, rs = k * (k + 1) / 2;
    for (int32_t r = 0; r < p->nrec; ++r) {
      const double wt = p->is_objective ? ow : w[p->rows[r]];
      double* o = out + p->hess_off + (size_t)r * rs;
      if (wt == 0.0) {
        for (int32_t s = 0; s < rs; ++s) o[s] = 0.0;
        continue;
      }
      gather(p, r, x, xl);
      int32_t slot = 0;
      for (int32_t j = 0; j < k; ++j) {
        for (int32_t f = 0; f < k; ++f) xd[f] = D2(xl[f], f == j ? 1.0 : 0.0);
        if (!fwd_dual(&p->tp, rec_reals(p, r), xd, vals)) { set_fail(fail, pid, r); return 0; }
        for (int32_t f = 0; f < k; ++f) xbar[f] = D1(0.0);
        rev_dual(&p->tp, vals, adj, D1(wt), xbar);
        for (int32_t i = j; i < k; ++i) {
          const double h = xbar[i].d;
          if (!isfinite(h)) { set_fail(fail, pid, r); return 0; }
          o[slot++] = h;
        }
      }
    }
    for (int64_t s = 0; s < p->ndbl; ++s) out[p->dbl[s]] += out[p->dbl[s]];
  }
  return 1;
}

/* ------------------------------------------------------------------ lifted */
/* lifted.hpp:25-100 (relative relaxation). */
void or_lifted_create(or_model* m, double relax, int64_t* sizes) {
  lifted_t* L = &m->lift;
  if (m->has_lifted) {
    free(L->free_of_full); free(L->full_of_free); free(L->jr); free(L->jc); free(L->jpick);
    free(L->hr); free(L->hc); free(L->hpick); free(L->sl); free(L->su);
  }
  m->has_lifted = 1;
  L->free_of_full = (int32_t*)malloc(sizeof(int32_t) * (m->n + 1));
  L->full_of_free = (int32_t*)malloc(sizeof(int32_t) * (m->n + 1));
  L->n_free = 0;
  for (int32_t i = 0; i < m->n; ++i) {
    if (m->xl[i] == m->xu[i]) {
      L->free_of_full[i] = -1;
    } else {
      L->free_of_full[i] = L->n_free;
      L->full_of_free[L->n_free++] = i;
    }
  }
  L->sl = (double*)malloc(sizeof(double) * (m->m + 1));
  L->su = (double*)malloc(sizeof(double) * (m->m + 1));
  for (int32_t i = 0; i < m->m; ++i) {
    const double lo = m->rl[i], hi = m->ru[i];
    if (lo == hi) {
      const double width = relax * fmax(1.0, fabs(lo));
      L->sl[i] = lo - width;
      L->su[i] = hi + width;
    } else {
      L->sl[i] = lo;
      L->su[i] = hi;
    }
  }
  L->jr = (int32_t*)malloc(sizeof(int32_t) * (m->nj + 1));
  L->jc = (int32_t*)malloc(sizeof(int32_t) * (m->nj + 1));
  L->jpick = (int32_t*)malloc(sizeof(int32_t) * (m->nj + 1));
  L->nj = 0;
  for (int64_t k = 0; k < m->nj; ++k) {
    const int32_t col = L->free_of_full[m->jc[k]];
    if (col < 0) continue;
    L->jr[L->nj] = m->jr[k];
    L->jc[L->nj] = col;
    L->jpick[L->nj] = (int32_t)k;
    L->nj++;
  }
  L->hr = (int32_t*)malloc(sizeof(int32_t) * (m->nh + 1));
  L->hc = (int32_t*)malloc(sizeof(int32_t) * (m->nh + 1));
  L->hpick = (int32_t*)malloc(sizeof(int32_t) * (m->nh + 1));
  L->nh = 0;
  for (int64_t k = 0; k < m->nh; ++k) {
    const int32_t r = L->free_of_full[m->hr[k]], c = L->free_of_full[m->hc[k]];
    if (r < 0 || c < 0) continue;
    L->hr[L->nh] = r;
    L->hc[L->nh] = c;
    L->hpick[L->nh] = (int32_t)k;
    L->nh++;
  }
  sizes[0] = L->n_free; sizes[1] = m->m; sizes[2] = L->nj; sizes[3] = L->nh;
}

void or_lifted_structure(const or_model* m, int32_t* free_to_full, int32_t* jr,
                         int32_t* jc, int32_t* hr, int32_t* hc, int32_t* jac_pick,
                         int32_t* hess_pick, double* sl, double* su) {
  const lifted_t* L = &m->lift;
  if (free_to_full) memcpy(free_to_full, L->full_of_free, sizeof(int32_t) * L->n_free);
  if (jr) memcpy(jr, L->jr, sizeof(int32_t) * L->nj);
  if (jc) memcpy(jc, L->jc, sizeof(int32_t) * L->nj);
  if (hr) memcpy(hr, L->hr, sizeof(int32_t) * L->nh);
  if (hc) memcpy(hc, L->hc, sizeof(int32_t) * L->nh);
  if (jac_pick) memcpy(jac_pick, L->jpick, sizeof(int32_t) * L->nj);
  if (hess_pick) memcpy(hess_pick, L->hpick, sizeof(int32_t) * L->nh);
  if (sl) memcpy(sl, L->sl, sizeof(double) * m->m);
  if (su) memcpy(su, L->su, sizeof(double) * m->m);
}

/* ------------------------------------------------------------------ sparse */
static int cmp_key(const void* a, const void* b, void* ctx) {
  const int64_t* key = (const int64_t*)ctx;
  const int64_t ka = key[*(const int64_t*)a], kb = key[*(const int64_t*)b];
  return ka < kb ? -1 : (ka > kb ? 1 : 0);
}

/* compress_to_csc (matrix.hpp:45-81): sort by (col,row), merge duplicates. */
static int32_t compress_csc(int32_t nrows, int32_t ncols, int64_t nnz, const int32_t* rows,
                            const int32_t* cols, int32_t* colptr, int32_t* rowidx,
                            int32_t* slot_map) {
  int64_t* key = (int64_t*)malloc(sizeof(int64_t) * (nnz + 1));
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (nnz + 1));
  for (int64_t k = 0; k < nnz; ++k) {
    key[k] = (int64_t)cols[k] * (int64_t)nrows + rows[k];
    order[k] = k;
  }
  qsort_r(order, (size_t)nnz, sizeof(int64_t), cmp_key, key);
  for (int32_t c = 0; c <= ncols; ++c) colptr[c] = 0;
  int32_t out = 0;
  int32_t last_c = -1, last_r = -1;
  for (int64_t i = 0; i < nnz; ++i) {
    const int64_t k = order[i];
    const int32_t c = cols[k], r = rows[k];
    if (c != last_c || r != last_r) {
      rowidx[out++] = r;
      colptr[c + 1]++;
      last_c = c;
      last_r = r;
    }
    slot_map[k] = out - 1;
  }
  for (int32_t c = 0; c < ncols; ++c) colptr[c + 1] += colptr[c];
  free(key);
  free(order);
  return out;
}

int32_t or_compress_to_csc(int32_t nrows, int32_t ncols, int64_t nnz, const int32_t* rows,
                           const int32_t* cols, int32_t* colptr, int32_t* rowidx,
                           int32_t* slot_map) {
  for (int64_t k = 0; k < nnz; ++k)
    if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols) return -1;
  return compress_csc(nrows, ncols, nnz, rows, cols, colptr, rowidx, slot_map);
}

/* --------------------------------------------------------------- condensed */
struct or_kkt {
  int32_t n, m;
  int64_t nj, nh, npair;
  int32_t *rowptr, *colidx, *jac_slots, annz;
  double* avals;
  int32_t *colptr, *rowidx, mnnz;
  int32_t *hess_slots, *pair_slots, *diag_slots;
  double* mvals;
};

/* condensed.hpp:29-90 */
or_kkt* or_kkt_create(int32_t n, int32_t m, int64_t nj, const int32_t* jr,
                      const int32_t* jc, int64_t nh, const int32_t* hr, const int32_t* hc) {
  or_kkt* K = (or_kkt*)calloc(1, sizeof(or_kkt));
  K->n = n; K->m = m; K->nj = nj; K->nh = nh;
  /* compress_to_csr = compress_to_csc of the transpose (matrix.hpp:83-97) */
  K->rowptr = (int32_t*)malloc(sizeof(int32_t) * (m + 1));
  K->colidx = (int32_t*)malloc(sizeof(int32_t) * (nj + 1));
  K->jac_slots = (int32_t*)malloc(sizeof(int32_t) * (nj + 1));
  K->annz = compress_csc(n, m, nj, jc, jr, K->rowptr, K->colidx, K->jac_slots);
  K->avals = (double*)calloc((size_t)K->annz + 1, sizeof(double));

  int64_t pc = 0;
  for (int32_t r = 0; r < m; ++r) {
    const int64_t len = K->rowptr[r + 1] - K->rowptr[r];
    pc += len * (len + 1) / 2;
  }
  K->npair = pc;
  const int64_t tot = nh + pc + n;
  int32_t* mr = (int32_t*)malloc(sizeof(int32_t) * (tot + 1));
  int32_t* mc = (int32_t*)malloc(sizeof(int32_t) * (tot + 1));
  int64_t q = 0;
  for (int64_t k = 0; k < nh; ++k) {
    mr[q] = hr[k] > hc[k] ? hr[k] : hc[k];
    mc[q] = hr[k] < hc[k] ? hr[k] : hc[k];
    ++q;
  }
  for (int32_t r = 0; r < m; ++r)
    for (int32_t ka = K->rowptr[r]; ka < K->rowptr[r + 1]; ++ka)
      for (int32_t kb = K->rowptr[r]; kb <= ka; ++kb) {
        mr[q] = K->colidx[ka];
        mc[q] = K->colidx[kb];
        ++q;
      }
  for (int32_t i = 0; i < n; ++i) { mr[q] = i; mc[q] = i; ++q; }
  int32_t* slots = (int32_t*)malloc(sizeof(int32_t) * (tot + 1));
  K->colptr = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  K->rowidx = (int32_t*)malloc(sizeof(int32_t) * (tot + 1));
  K->mnnz = compress_csc(n, n, tot, mr, mc, K->colptr, K->rowidx, slots);
  K->hess_slots = (int32_t*)malloc(sizeof(int32_t) * (nh + 1));
  K->pair_slots = (int32_t*)malloc(sizeof(int32_t) * (pc + 1));
  K->diag_slots = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  memcpy(K->hess_slots, slots, sizeof(int32_t) * nh);
  memcpy(K->pair_slots, slots + nh, sizeof(int32_t) * pc);
  memcpy(K->diag_slots, slots + nh + pc, sizeof(int32_t) * n);
  K->mvals = (double*)calloc((size_t)K->mnnz + 1, sizeof(double));
  free(mr); free(mc); free(slots);
  return K;
}

or_kkt* or_kkt_create_model(or_model* m) {
  const lifted_t* L = &m->lift;
  return or_kkt_create(L->n_free, m->m, L->nj, L->jr, L->jc, L->nh, L->hr, L->hc);
}

void or_kkt_free(or_kkt* K) {
  if (!K) return;
  free(K->rowptr); free(K->colidx); free(K->jac_slots); free(K->avals);
  free(K->colptr); free(K->rowidx); free(K->hess_slots); free(K->pair_slots);
  free(K->diag_slots); free(K->mvals);
  free(K);
}

void or_kkt_sizes(const or_kkt* K, int64_t* s) {
  s[0] = K->n; s[1] = K->annz; s[2] = K->mnnz; s[3] = K->npair;
}

void or_kkt_structure(const or_kkt* K, int32_t* rowptr, int32_t* colidx, int32_t* colptr,
                      int32_t* rowidx) {
  if (rowptr) memcpy(rowptr, K->rowptr, sizeof(int32_t) * (K->m + 1));
  if (colidx) memcpy(colidx, K->colidx, sizeof(int32_t) * K->annz);
  if (colptr) memcpy(colptr, K->colptr, sizeof(int32_t) * (K->n + 1));
  if (rowidx) memcpy(rowidx, K->rowidx, sizeof(int32_t) * K->mnnz);
}

void or_kkt_slots(const or_kkt* K, int32_t* jac_slots, int32_t* hess_slots,
                  int32_t* pair_slots, int32_t* diag_slots) {
  if (jac_slots) memcpy(jac_slots, K->jac_slots, sizeof(int32_t) * K->nj);
  if (hess_slots) memcpy(hess_slots, K->hess_slots, sizeof(int32_t) * K->nh);
  if (pair_slots) memcpy(pair_slots, K->pair_slots, sizeof(int32_t) * K->npair);
  if (diag_slots) memcpy(diag_slots, K->diag_slots, sizeof(int32_t) * K->n);
}

/* set_jacobian -> scatter_values (condensed.hpp:99-101, matrix.hpp:100-106) */
void or_kkt_set_jacobian(or_kkt* K, const double* jvals) {
  for (int32_t i = 0; i < K->annz; ++i) K->avals[i] = 0.0;
  for (int64_t k = 0; k < K->nj; ++k) K->avals[K->jac_slots[k]] += jvals[k];
}

/* assemble (condensed.hpp:105-135) */
void or_kkt_assemble(or_kkt* K, const double* hvals, const double* sx, const double* ss,
                     double dw, double dc) {
  double* dvec = (double*)malloc(sizeof(double) * (K->m + 1));
  for (int32_t i = 0; i < K->m; ++i) {
    const double sd = ss[i] + dw;
    const double c = 1.0 / (1.0 + dc * sd);
    dvec[i] = sd * c;
  }
  for (int32_t i = 0; i < K->mnnz; ++i) K->mvals[i] = 0.0;
  for (int64_t k = 0; k < K->nh; ++k) K->mvals[K->hess_slots[k]] += hvals[k];
  int64_t p = 0;
  for (int32_t r = 0; r < K->m; ++r) {
    const double w = dvec[r];
    for (int32_t ka = K->rowptr[r]; ka < K->rowptr[r + 1]; ++ka) {
      const double va = w * K->avals[ka];
      for (int32_t kb = K->rowptr[r]; kb <= ka; ++kb, ++p)
        K->mvals[K->pair_slots[p]] += va * K->avals[kb];
    }
  }
  for (int32_t i = 0; i < K->n; ++i) K->mvals[K->diag_slots[i]] += dw + sx[i];
  free(dvec);
}

void or_kkt_values(const or_kkt* K, double* a_vals, double* m_vals) {
  if (a_vals) memcpy(a_vals, K->avals, sizeof(double) * K->annz);
  if (m_vals) memcpy(m_vals, K->mvals, sizeof(double) * K->mnnz);
}
