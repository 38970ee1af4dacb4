"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU checkers.

* `OracleModel` / `OracleKkt`: the plain-C restatement (oracle/gn_oracle.c,
  built into oracle/_build/libgn_oracle.so).
* `RefModel`: the UNMODIFIED reference compiled from /root/reference by
  oracle/Makefile into oracle/_ref/libgridnlp_ref.so (present wherever
  build() ran with /root/reference available; it travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "_build" / "libgn_oracle.so"
REF_LIB = HERE / "_ref" / "libgridnlp_ref.so"

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


def _f(a):
    return None if a is None else a.ctypes.data_as(f64p)


def _i(a):
    return None if a is None else a.ctypes.data_as(i32p)


_or = None
_ref = None


def oracle_lib():
    global _or
    if _or is None:
        if not ORACLE_LIB.exists():
            raise ImportError(f"{ORACLE_LIB} missing; run make -C oracle")
        L = C.CDLL(str(ORACLE_LIB))
        sig = {
            "or_model_create": (vp, [vp, C.c_int32, f64p, C.c_char_p, C.c_int]),
            "or_model_free": (None, [vp]),
            "or_model_sizes": (None, [vp, i64p]),
            "or_model_bounds": (None, [vp, f64p, f64p, f64p, f64p, f64p]),
            "or_model_structure": (None, [vp, i32p, i32p, i32p, i32p]),
            "or_model_offsets": (None, [vp, i64p, i64p, i64p]),
            "or_eval_f": (C.c_int, [vp, f64p, f64p, i32p]),
            "or_eval_grad": (C.c_int, [vp, f64p, f64p, i32p]),
            "or_eval_g": (C.c_int, [vp, f64p, f64p, i32p]),
            "or_eval_jac": (C.c_int, [vp, f64p, f64p, i32p]),
            "or_eval_hess": (C.c_int, [vp, f64p, f64p, C.c_double, f64p, i32p]),
            "or_lifted_create": (None, [vp, C.c_double, i64p]),
            "or_lifted_structure": (None, [vp, i32p, i32p, i32p, i32p, i32p, i32p, i32p, f64p,
                                           f64p]),
            "or_kkt_create": (vp, [C.c_int32, C.c_int32, C.c_int64, i32p, i32p, C.c_int64, i32p,
                                   i32p]),
            "or_kkt_create_model": (vp, [vp]),
            "or_kkt_free": (None, [vp]),
            "or_kkt_sizes": (None, [vp, i64p]),
            "or_kkt_structure": (None, [vp, i32p, i32p, i32p, i32p]),
            "or_kkt_slots": (None, [vp, i32p, i32p, i32p, i32p]),
            "or_kkt_set_jacobian": (None, [vp, f64p]),
            "or_kkt_assemble": (None, [vp, f64p, f64p, f64p, C.c_double, C.c_double]),
            "or_kkt_values": (None, [vp, f64p, f64p]),
            "or_compress_to_csc": (C.c_int32, [C.c_int32, C.c_int32, C.c_int64, i32p, i32p,
                                               i32p, i32p, i32p]),
        }
        for k, (r, a) in sig.items():
            getattr(L, k).restype = r
            getattr(L, k).argtypes = a
        _or = L
    return _or


def ref_available() -> bool:
    return REF_LIB.exists()


f64pp = C.POINTER(C.POINTER(C.c_double))


def _pp(arrays):
    """double*[k] over float64 numpy arrays (kept alive by the caller)."""
    return (C.POINTER(C.c_double) * len(arrays))(*[_f(a) for a in arrays])


def ref_lib():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise ImportError(f"{REF_LIB} missing; run make -C oracle ref (needs /root/reference)")
        L = C.CDLL(str(REF_LIB))
        sig = {
            "gnr_net_parse": (vp, [C.c_char_p, C.c_double, C.c_char_p, C.c_int]),
            "gnr_net_free": (None, [vp]),
            "gnr_net_dims": (None, [vp, i32p]),
            "gnr_net_export": (None, [vp, f64p] + [f64p] * 4 + [i32p, i32p] + [f64p] * 5
                               + [i32p] + [f64p] * 10 + [i32p, f64p, f64p]),
            "gnr_load_profile": (None, [vp, C.c_int32, C.c_double, C.c_uint64, C.c_double,
                                        C.c_double, f64p]),
            "gnr_model_create": (vp, [vp, C.c_int32, f64p, C.c_char_p, C.c_int]),
            "gnr_model_free": (None, [vp]),
            "gnr_model_set_threads": (None, [vp, C.c_int]),
            "gnr_model_sizes": (None, [vp, i64p]),
            "gnr_model_bounds": (None, [vp, f64p, f64p, f64p, f64p, f64p]),
            "gnr_model_structure": (None, [vp, i32p, i32p, i32p, i32p]),
            "gnr_eval_f": (C.c_int, [vp, f64p, f64p, i32p]),
            "gnr_eval_grad": (C.c_int, [vp, f64p, f64p, i32p]),
            "gnr_eval_g": (C.c_int, [vp, f64p, f64p, i32p]),
            "gnr_eval_jac": (C.c_int, [vp, f64p, f64p, i32p]),
            "gnr_eval_hess": (C.c_int, [vp, f64p, f64p, C.c_double, f64p, i32p]),
            "gnr_lifted_create": (None, [vp, C.c_double, i64p]),
            "gnr_lifted_structure": (None, [vp, i32p, i32p, i32p, i32p, i32p, f64p, f64p]),
            "gnr_lifted_eval_jac": (C.c_int, [vp, f64p, f64p]),
            "gnr_lifted_eval_hess": (C.c_int, [vp, f64p, f64p, C.c_double, f64p]),
            "gnr_kkt_create": (None, [vp, i64p]),
            "gnr_kkt_structure": (None, [vp, i32p, i32p, i32p, i32p]),
            "gnr_kkt_set_jacobian": (None, [vp, f64p]),
            "gnr_kkt_assemble": (None, [vp, f64p, f64p, f64p, C.c_double, C.c_double]),
            "gnr_kkt_values": (None, [vp, f64p, f64p]),
            "gnr_compress_to_csc": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, i32p, i32p,
                                              i32p, i32p, i32p]),
            "gnr_solve": (None, [vp, C.c_double, C.c_int, f64p]),
            "gnr_lifted_bounds": (None, [vp, f64p, f64p, f64p, f64p]),
            "gnr_ipm_jac_t": (None, [vp, f64p, f64p, f64p]),
            "gnr_ipm_jac": (None, [vp, f64p, f64p, f64p]),
            "gnr_ipm_residuals": (None, [vp, f64pp, f64pp, f64p, f64p, f64p, C.c_double, f64pp]),
            "gnr_ipm_condense": (None, [vp, f64pp, f64pp, f64pp, f64p, f64p, f64p, f64p]),
            "gnr_ipm_ftb": (None, [vp, f64pp, f64pp, f64pp, C.c_double, f64p]),
            "gnr_ipm_barrier": (C.c_double, [vp, f64pp, C.c_double, f64p, f64p, C.c_double]),
            "gnr_ipm_slope": (C.c_double, [vp, f64pp, f64p, f64pp, f64pp, C.c_double]),
            "gnr_ipm_violation": (C.c_double, [vp, f64p, f64p]),
            "gnr_ipm_kkt_error": (None, [vp, f64pp, f64pp, f64pp, C.c_double, f64p]),
            "gnr_ipm_recover": (None, [vp, f64pp, f64pp, f64pp, f64pp, f64pp]),
            "gnr_kkt_solve_parts": (None, [vp, f64p, f64p, f64p, f64p, C.c_double, C.c_double,
                                           f64p, f64p, f64p, f64p]),
        }
        for k, (r, a) in sig.items():
            getattr(L, k).restype = r
            getattr(L, k).argtypes = a
        _ref = L
    return _ref


# ------------------------------------------------------------------ networks
def ref_parse_matpower(text: str, ramp_fraction: float = 0.1):
    """Parse MATPOWER text with the reference parser; returns a Network."""
    from paper_2405_14032_b200.network import Network
    L = ref_lib()
    err = C.create_string_buffer(512)
    h = L.gnr_net_parse(text.encode(), ramp_fraction, err, 512)
    if not h:
        raise ValueError(err.value.decode())
    try:
        d = (C.c_int32 * 5)()
        L.gnr_net_dims(h, d)
        N, Ln, G, D, ref = list(d)
        base = np.zeros(1)
        bus = [np.empty(N) for _ in range(4)]
        li = [np.empty(Ln, np.int32) for _ in range(2)]
        lf = [np.empty(Ln) for _ in range(5)]
        gb = np.empty(G, np.int32)
        gf = [np.empty(G) for _ in range(10)]
        db = np.empty(D, np.int32)
        dfl = [np.empty(D) for _ in range(2)]
        L.gnr_net_export(h, _f(base), *map(_f, bus), *map(_i, li), *map(_f, lf), _i(gb),
                         *map(_f, gf), _i(db), *map(_f, dfl))
        return Network(base_mva=float(base[0]), reference_bus=ref,
                       bus_vmin=bus[0], bus_vmax=bus[1], vm_start=bus[2], va_start=bus[3],
                       line_from=li[0], line_to=li[1], line_g=lf[0], line_b=lf[1],
                       line_smax=lf[2], line_amin=lf[3], line_amax=lf[4], gen_bus=gb,
                       gen_pmin=gf[0], gen_pmax=gf[1], gen_qmin=gf[2], gen_qmax=gf[3],
                       gen_ramp=gf[4], gen_c2=gf[5], gen_c1=gf[6], gen_c0=gf[7],
                       gen_pstart=gf[8], gen_qstart=gf[9], load_bus=db, load_p=dfl[0],
                       load_q=dfl[1])
    finally:
        L.gnr_net_free(h)


def _ref_net_handle(net):
    """Reference NetworkData from a Network (via MATPOWER-free export path)."""
    # The reference parser is the only public way to build NetworkData from
    # arrays without writing C++; emit an equivalent MATPOWER text instead.
    raise NotImplementedError


class _ModelBase:
    def _sz(self):
        return self.sizes  # [n, m, jnnz, hnnz, LT, GR]

    def bounds(self):
        n, m = self.sizes[0], self.sizes[1]
        xl, xu, xs = np.empty(n), np.empty(n), np.empty(n)
        rl, ru = np.empty(m), np.empty(m)
        self._bounds(self.h, _f(xl), _f(xu), _f(xs), _f(rl), _f(ru))
        return xl, xu, xs, rl, ru

    def structure(self):
        nj, nh = self.sizes[2], self.sizes[3]
        jr, jc = np.empty(nj, np.int32), np.empty(nj, np.int32)
        hr, hc = np.empty(nh, np.int32), np.empty(nh, np.int32)
        self._structure(self.h, _i(jr), _i(jc), _i(hr), _i(hc))
        return jr, jc, hr, hc

    def _ev(self, fn, x, size, *extra):
        out = np.empty(max(size, 1))
        fail = np.full(2, -1, np.int32)
        ok = fn(self.h, _f(np.ascontiguousarray(x, np.float64)), *extra, _f(out), _i(fail))
        return bool(ok), out[:size], (int(fail[0]), int(fail[1]))

    def eval_f(self, x):
        ok, out, fail = self._ev(self._f, x, 1)
        return ok, float(out[0]), fail

    def eval_grad(self, x):
        return self._ev(self._grad, x, self.sizes[0])

    def eval_g(self, x):
        return self._ev(self._g, x, self.sizes[1])

    def eval_jac(self, x):
        return self._ev(self._jac, x, self.sizes[2])

    def eval_hess(self, x, w, ow):
        return self._ev(self._hess, x, self.sizes[3], _f(np.ascontiguousarray(w, np.float64)),
                        float(ow))


class OracleModel(_ModelBase):
    """The C restatement of build_multiperiod_opf + PatternModel (oracle/gn_oracle.c)."""

    def __init__(self, net, periods: int, scale: np.ndarray):
        L = oracle_lib()
        self.L = L
        self._cnet = net.to_c()
        self._scale = np.ascontiguousarray(scale, np.float64).reshape(-1)
        err = C.create_string_buffer(256)
        self.h = L.or_model_create(C.byref(self._cnet), periods, _f(self._scale), err, 256)
        if not self.h:
            raise ValueError(err.value.decode())
        s = (C.c_int64 * 6)()
        L.or_model_sizes(self.h, s)
        self.sizes = list(s)
        self._bounds, self._structure = L.or_model_bounds, L.or_model_structure
        self._f, self._grad, self._g = L.or_eval_f, L.or_eval_grad, L.or_eval_g
        self._jac, self._hess = L.or_eval_jac, L.or_eval_hess

    def __del__(self):
        if getattr(self, "h", None):
            self.L.or_model_free(self.h)
            self.h = None

    def offsets(self):
        a, b, c = (C.c_int64 * 12)(), (C.c_int64 * 12)(), (C.c_int64 * 12)()
        self.L.or_model_offsets(self.h, a, b, c)
        return list(a), list(b), list(c)

    def lift(self, relax: float):
        s = (C.c_int64 * 4)()
        self.L.or_lifted_create(self.h, relax, s)
        n, m, nj, nh = list(s)
        self.lifted_sizes = (n, m, nj, nh)
        f2f = np.empty(n, np.int32)
        jr, jc, jp = (np.empty(nj, np.int32) for _ in range(3))
        hr, hc, hp = (np.empty(nh, np.int32) for _ in range(3))
        sl, su = np.empty(m), np.empty(m)
        self.L.or_lifted_structure(self.h, _i(f2f), _i(jr), _i(jc), _i(hr), _i(hc), _i(jp),
                                   _i(hp), _f(sl), _f(su))
        return dict(free_to_full=f2f, jac_rows=jr, jac_cols=jc, jac_pick=jp, hess_rows=hr,
                    hess_cols=hc, hess_pick=hp, s_lower=sl, s_upper=su)

    def kkt(self):
        return OracleKkt(h=self.L.or_kkt_create_model(self.h), owner=self)


class OracleKkt:
    def __init__(self, n=None, m=None, jr=None, jc=None, hr=None, hc=None, h=None, owner=None):
        L = oracle_lib()
        self.L = L
        self._owner = owner
        if h is None:
            jr, jc = np.ascontiguousarray(jr, np.int32), np.ascontiguousarray(jc, np.int32)
            hr, hc = np.ascontiguousarray(hr, np.int32), np.ascontiguousarray(hc, np.int32)
            h = L.or_kkt_create(n, m, len(jr), _i(jr), _i(jc), len(hr), _i(hr), _i(hc))
            self.m = m
        self.h = h
        s = (C.c_int64 * 4)()
        L.or_kkt_sizes(h, s)
        self.dim, self.a_nnz, self.m_nnz, self.pair_count = list(s)
        if owner is not None:
            self.m = owner.sizes[1]
            self.nj, self.nh = owner.lifted_sizes[2], owner.lifted_sizes[3]
        else:
            self.nj, self.nh = len(jr), len(hr)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.or_kkt_free(self.h)
            self.h = None

    def structure(self):
        rp = np.empty(self.m + 1, np.int32)
        ci = np.empty(self.a_nnz, np.int32)
        cp = np.empty(self.dim + 1, np.int32)
        ri = np.empty(self.m_nnz, np.int32)
        self.L.or_kkt_structure(self.h, _i(rp), _i(ci), _i(cp), _i(ri))
        return rp, ci, cp, ri

    def slots(self):
        js = np.empty(self.nj, np.int32)
        hs = np.empty(self.nh, np.int32)
        ps = np.empty(self.pair_count, np.int32)
        ds = np.empty(self.dim, np.int32)
        self.L.or_kkt_slots(self.h, _i(js), _i(hs), _i(ps), _i(ds))
        return js, hs, ps, ds

    def set_jacobian(self, j):
        self.L.or_kkt_set_jacobian(self.h, _f(np.ascontiguousarray(j, np.float64)))

    def assemble(self, h, sx, ss, dw, dc):
        self.L.or_kkt_assemble(self.h, _f(np.ascontiguousarray(h, np.float64)),
                               _f(np.ascontiguousarray(sx, np.float64)),
                               _f(np.ascontiguousarray(ss, np.float64)), dw, dc)

    def values(self):
        a, m = np.empty(self.a_nnz), np.empty(self.m_nnz)
        self.L.or_kkt_values(self.h, _f(a), _f(m))
        return a, m


def oracle_compress_to_csc(nrows, ncols, rows, cols):
    rows = np.ascontiguousarray(rows, np.int32)
    cols = np.ascontiguousarray(cols, np.int32)
    cp = np.empty(ncols + 1, np.int32)
    ri = np.empty(max(len(rows), 1), np.int32)
    sm = np.empty(max(len(rows), 1), np.int32)
    nnz = oracle_lib().or_compress_to_csc(nrows, ncols, len(rows), _i(rows), _i(cols), _i(cp),
                                          _i(ri), _i(sm))
    if nnz < 0:
        raise ValueError("compress_to_csc: coordinate out of range")
    return cp, ri[:nnz], sm[: len(rows)]


class RefModel(_ModelBase):
    """The compiled reference (oracle/_ref): build_multiperiod_opf + PatternModel."""

    def __init__(self, matpower_text: str, periods: int, scale: np.ndarray,
                 ramp_fraction: float = 0.1):
        L = ref_lib()
        self.L = L
        err = C.create_string_buffer(512)
        self.net = L.gnr_net_parse(matpower_text.encode(), ramp_fraction, err, 512)
        if not self.net:
            raise ValueError(err.value.decode())
        self._scale = np.ascontiguousarray(scale, np.float64).reshape(-1)
        self.h = L.gnr_model_create(self.net, periods, _f(self._scale), err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        s = (C.c_int64 * 6)()
        L.gnr_model_sizes(self.h, s)
        self.sizes = list(s)
        self._bounds, self._structure = L.gnr_model_bounds, L.gnr_model_structure
        self._f, self._grad, self._g = L.gnr_eval_f, L.gnr_eval_grad, L.gnr_eval_g
        self._jac, self._hess = L.gnr_eval_jac, L.gnr_eval_hess

    def __del__(self):
        if getattr(self, "h", None):
            self.L.gnr_model_free(self.h)
            self.h = None
        if getattr(self, "net", None):
            self.L.gnr_net_free(self.net)
            self.net = None

    def set_threads(self, n: int):
        self.L.gnr_model_set_threads(self.h, n)

    def lift(self, relax: float):
        s = (C.c_int64 * 4)()
        self.L.gnr_lifted_create(self.h, relax, s)
        n, m, nj, nh = list(s)
        self.lifted_sizes = (n, m, nj, nh)
        f2f = np.empty(n, np.int32)
        jr, jc = np.empty(nj, np.int32), np.empty(nj, np.int32)
        hr, hc = np.empty(nh, np.int32), np.empty(nh, np.int32)
        sl, su = np.empty(m), np.empty(m)
        self.L.gnr_lifted_structure(self.h, _i(f2f), _i(jr), _i(jc), _i(hr), _i(hc), _f(sl),
                                    _f(su))
        return dict(free_to_full=f2f, jac_rows=jr, jac_cols=jc, hess_rows=hr, hess_cols=hc,
                    s_lower=sl, s_upper=su)

    def kkt_create(self):
        s = (C.c_int64 * 4)()
        self.L.gnr_kkt_create(self.h, s)
        self.kkt_sizes = list(s)  # dim, a_nnz, m_nnz, factor_nnz
        return self.kkt_sizes

    def kkt_structure(self):
        dim, annz, mnnz, _ = self.kkt_sizes
        rp = np.empty(self.sizes[1] + 1, np.int32)
        ci = np.empty(annz, np.int32)
        cp = np.empty(dim + 1, np.int32)
        ri = np.empty(mnnz, np.int32)
        self.L.gnr_kkt_structure(self.h, _i(rp), _i(ci), _i(cp), _i(ri))
        return rp, ci, cp, ri

    def kkt_set_jacobian(self, jl):
        self.L.gnr_kkt_set_jacobian(self.h, _f(np.ascontiguousarray(jl, np.float64)))

    def kkt_assemble(self, hl, sx, ss, dw, dc):
        self.L.gnr_kkt_assemble(self.h, _f(np.ascontiguousarray(hl, np.float64)),
                                _f(np.ascontiguousarray(sx, np.float64)),
                                _f(np.ascontiguousarray(ss, np.float64)), dw, dc)

    def kkt_values(self):
        a = np.empty(self.kkt_sizes[1])
        m = np.empty(self.kkt_sizes[2])
        self.L.gnr_kkt_values(self.h, _f(a), _f(m))
        return a, m

    # ---- ipm/iterate.hpp vector ops on the lifted problem (arrays in the
    # Iterate / Residuals / Direction field order x s y zlx zux zls zus)
    def lifted_bounds(self):
        n, m = self.lifted_sizes[0], self.lifted_sizes[1]
        b = [np.empty(n), np.empty(n), np.empty(m), np.empty(m)]
        self.L.gnr_lifted_bounds(self.h, *[_f(a) for a in b])
        return b

    def ipm_jac_t(self, jv, y):
        out = np.empty(self.lifted_sizes[0])
        self.L.gnr_ipm_jac_t(self.h, _f(jv), _f(y), _f(out))
        return out

    def ipm_jac(self, jv, x):
        out = np.empty(self.lifted_sizes[1])
        self.L.gnr_ipm_jac(self.h, _f(jv), _f(x), _f(out))
        return out

    def _nm(self):
        n, m = self.lifted_sizes[0], self.lifted_sizes[1]
        return [n, m, m, n, n, m, m]

    def ipm_residuals(self, bounds, it, grad, g, jv, mu):
        out = [np.empty(k) for k in self._nm()]
        self.L.gnr_ipm_residuals(self.h, _pp(bounds), _pp(it), _f(grad), _f(g), _f(jv), mu,
                                 _pp(out))
        return out

    def ipm_condense(self, bounds, it, r):
        n, m = self.lifted_sizes[0], self.lifted_sizes[1]
        o = [np.empty(n), np.empty(m), np.empty(n), np.empty(m)]
        self.L.gnr_ipm_condense(self.h, _pp(bounds), _pp(it), _pp(r), *[_f(a) for a in o])
        return o

    def ipm_ftb(self, bounds, it, d, tau):
        out = np.empty(2)
        self.L.gnr_ipm_ftb(self.h, _pp(bounds), _pp(it), _pp(d), tau, _f(out))
        return out

    def ipm_barrier(self, bounds, f, x, s, mu):
        return self.L.gnr_ipm_barrier(self.h, _pp(bounds), f, _f(x), _f(s), mu)

    def ipm_slope(self, bounds, grad, it, d, mu):
        return self.L.gnr_ipm_slope(self.h, _pp(bounds), _f(grad), _pp(it), _pp(d), mu)

    def ipm_violation(self, g, s):
        return self.L.gnr_ipm_violation(self.h, _f(g), _f(s))

    def ipm_kkt_error(self, bounds, it, r, mu):
        out = np.empty(3)
        self.L.gnr_ipm_kkt_error(self.h, _pp(bounds), _pp(it), _pp(r), mu, _f(out))
        return out

    def ipm_recover(self, bounds, it, r, d):
        n, m = self.lifted_sizes[0], self.lifted_sizes[1]
        o = [np.empty(n), np.empty(n), np.empty(m), np.empty(m)]
        self.L.gnr_ipm_recover(self.h, _pp(bounds), _pp(it), _pp(r), _pp(d), _pp(o))
        return o

    def kkt_solve_parts(self, qx, qs, qy, ss, dw, dc, dx):
        n, m = self.lifted_sizes[0], self.lifted_sizes[1]
        rhs, ds, dy = np.empty(n), np.empty(m), np.empty(m)
        self.L.gnr_kkt_solve_parts(self.h, _f(qx), _f(qs), _f(qy), _f(ss), dw, dc, _f(dx),
                                   _f(rhs), _f(ds), _f(dy))
        return rhs, ds, dy

    def solve(self, tol=1e-4, max_iter=500):
        out = np.zeros(5)
        self.L.gnr_solve(self.h, tol, max_iter, _f(out))
        return dict(iterations=int(out[0]), objective=float(out[1]), status=int(out[2]),
                    restorations=int(out[3]), seconds=float(out[4]))


def ref_load_profile(matpower_text: str, T: int, resolution=60.0, seed=1, amplitude=0.2,
                     noise=0.02, ramp_fraction=0.1):
    L = ref_lib()
    err = C.create_string_buffer(512)
    h = L.gnr_net_parse(matpower_text.encode(), ramp_fraction, err, 512)
    if not h:
        raise ValueError(err.value.decode())
    try:
        d = (C.c_int32 * 5)()
        L.gnr_net_dims(h, d)
        out = np.empty(T * max(d[3], 1))
        L.gnr_load_profile(h, T, resolution, seed, amplitude, noise, _f(out))
        return out[: T * d[3]].reshape(T, d[3])
    finally:
        L.gnr_net_free(h)


DROPIN = HERE / "_ref" / "ipm_dropin"


def write_network_bin(path, net, T, scale):
    """The binary network file of oracle/ipm_dropin.cpp (its load())."""
    with open(path, "wb") as f:
        np.array([net.n_bus, net.n_line, net.n_gen, net.n_load, net.reference_bus, T],
                 np.int32).tofile(f)
        np.array([net.base_mva], np.float64).tofile(f)
        for k in ("bus_vmin", "bus_vmax", "vm_start", "va_start"):
            getattr(net, k).tofile(f)
        net.line_from.tofile(f)
        net.line_to.tofile(f)
        for k in ("line_g", "line_b", "line_smax", "line_amin", "line_amax"):
            getattr(net, k).tofile(f)
        net.gen_bus.tofile(f)
        for k in ("gen_pmin", "gen_pmax", "gen_qmin", "gen_qmax", "gen_ramp", "gen_c2", "gen_c1",
                  "gen_c0", "gen_pstart", "gen_qstart", "gen_qstart"):
            getattr(net, k).tofile(f)
        net.load_bus.tofile(f)
        net.load_p.tofile(f)
        net.load_q.tofile(f)
        np.ascontiguousarray(scale, np.float64).tofile(f)
