"""Python mirror of the reference interfaces over the C-ABI (test/bench host).

`OpfNlp` mirrors ipm::PatternNlp / NlpProblem (ipm/nlp.hpp:15-39,
ipm/pattern_nlp.hpp:15-62): the same method names, the same argument meaning,
and the same error behaviour (construction mistakes raise, evaluation
failures return False and are described by `last_failure`).  `CondensedKkt`
mirrors ipm::CondensedKkt (ipm/condensed.hpp:27-185) minus factorize/solve.

Arrays may be numpy (host mode: GN_MEM_HOST) or CUDA torch tensors / raw
device pointers (device mode).  Every call goes to the CUDA library; there is
no CPU path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from .abi import GN_IN_FULL, GN_MEM_DEVICE, GN_MEM_DEVICE_ASYNC, GN_MEM_HOST, GnError, GnSizes
from .network import Network


class GridError(RuntimeError):
    """A construction/shape error (the reference throws gridnlp::Error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _check(rc: int, err: GnError | None = None, what: str = ""):
    if rc != abi.GN_OK:
        msg = err.message.decode() if err is not None else ""
        raise GridError(rc, f"{what}: {msg} (code {rc})")


def _f64(a):
    """Pointer for a float64 numpy array, CUDA tensor, or int device address."""
    if a is None:
        return None
    if isinstance(a, int):
        return C.cast(C.c_void_p(a), abi.f64p)
    if hasattr(a, "data_ptr"):
        return C.cast(C.c_void_p(a.data_ptr()), abi.f64p)
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(abi.f64p)


def _i32(a):
    if a is None:
        return None
    if isinstance(a, int):
        return C.cast(C.c_void_p(a), abi.i32p)
    if hasattr(a, "data_ptr"):
        return C.cast(C.c_void_p(a.data_ptr()), abi.i32p)
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(abi.i32p)


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy (driver_types.h)


def _stream_arg(handle: int) -> int:
    """torch's default stream (handle 0) is the legacy default stream; the C-ABI's NULL
    means "reset to the object's own stream", so it is passed as cudaStreamLegacy."""
    return CUDA_STREAM_LEGACY if int(handle) == 0 else int(handle)


def load_profile(n_load: int, periods: int, resolution: float = 60.0, seed: int = 1,
                 amplitude: float = 0.2, noise: float = 0.02) -> np.ndarray:
    """generate_load_profile (network.hpp:104-140), T x n_load, bit-identical."""
    out = np.empty(periods * max(n_load, 1), dtype=np.float64)
    err = GnError()
    _check(abi.lib().gn_load_profile(n_load, periods, resolution, seed, amplitude, noise,
                                     _f64(out), C.byref(err)), err, "load profile")
    return out[: periods * n_load].reshape(periods, n_load)


class OpfNlp:
    """Multi-period OPF on one B200 — the NlpProblem the reference's PatternNlp exposes."""

    def __init__(self, net: Network, periods: int, scale: np.ndarray, device: int = 0,
                 shard: tuple[int, int] | None = None):
        """shard = (periods_total, first_period): this object is the period shard
        [first_period, first_period + periods) of a periods_total horizon
        (gn_ctx_create_shard); scale is that slice of the demand table."""
        self.lib = abi.lib()
        self.net = net
        self._cnet = net.to_c()
        self._scale = np.ascontiguousarray(scale, dtype=np.float64).reshape(-1)
        if self._scale.size != periods * net.n_load:
            raise GridError(abi.GN_ERR_INVALID, "opf: load profile does not match network loads")
        h = C.c_void_p()
        err = GnError()
        if shard is None:
            rc = self.lib.gn_ctx_create(C.byref(self._cnet), periods, _f64(self._scale), device,
                                        C.byref(h), C.byref(err))
        else:
            rc = self.lib.gn_ctx_create_shard(C.byref(self._cnet), shard[0], shard[1], periods,
                                              _f64(self._scale), device, C.byref(h), C.byref(err))
        _check(rc, err, "gn_ctx_create")
        self.h = h
        self.device = device
        self.last_failure = ""
        self.last_error = (-1, -1)
        self._sizes()

    def _sizes(self):
        s = GnSizes()
        self.lib.gn_ctx_sizes(self.h, C.byref(s))
        self.sizes = s
        return s

    def close(self):
        if getattr(self, "h", None):
            self.lib.gn_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- NlpProblem sizes / bounds / structure (nlp.hpp:19-30)
    def n_vars(self) -> int:
        return self.sizes.n_vars

    def n_cons(self) -> int:
        return self.sizes.n_cons

    def bounds(self):
        n, m = self.n_vars(), self.n_cons()
        xl, xu, xs = (np.empty(n) for _ in range(3))
        rl, ru = np.empty(m), np.empty(m)
        _check(self.lib.gn_ctx_bounds(self.h, _f64(xl), _f64(xu), _f64(xs), _f64(rl), _f64(ru)))
        return xl, xu, xs, rl, ru

    def x_lower(self):
        return self.bounds()[0]

    def x_upper(self):
        return self.bounds()[1]

    def x_start(self):
        return self.bounds()[2]

    def row_lower(self):
        return self.bounds()[3]

    def row_upper(self):
        return self.bounds()[4]

    def jac_structure(self):
        nj = self.sizes.jac_nnz
        r, c = np.empty(nj, np.int32), np.empty(nj, np.int32)
        _check(self.lib.gn_jac_structure(self.h, _i32(r), _i32(c), GN_MEM_HOST))
        return r, c

    def hess_structure(self):
        nh = self.sizes.hess_nnz
        r, c = np.empty(nh, np.int32), np.empty(nh, np.int32)
        _check(self.lib.gn_hess_structure(self.h, _i32(r), _i32(c), GN_MEM_HOST))
        return r, c

    # ---- callbacks (nlp.hpp:32-38).  Host numpy in/out; returns bool.
    def _record(self, rc: int, err: GnError) -> bool:
        if rc == abi.GN_ERR_EVAL:
            self.last_failure = err.message.decode()
            self.last_error = (err.pattern, err.record)
            return False
        _check(rc, err, "evaluation")
        return True

    def eval_f(self, x: np.ndarray, out=None):
        out = np.zeros(1) if out is None else out
        err = GnError()
        ok = self._record(self.lib.gn_eval_f(self.h, _f64(x), _f64(out), GN_MEM_HOST,
                                             C.byref(err)), err)
        return ok, float(out[0])

    def _eval_vec(self, fn, x, size, *extra, out=None):
        out = np.empty(size) if out is None else out
        err = GnError()
        ok = self._record(fn(self.h, _f64(x), *extra, _f64(out), GN_MEM_HOST, C.byref(err)), err)
        return ok, out

    def eval_grad(self, x, out=None):
        return self._eval_vec(self.lib.gn_eval_grad, x, self.n_vars(), out=out)

    def eval_g(self, x, out=None):
        return self._eval_vec(self.lib.gn_eval_g, x, self.n_cons(), out=out)

    def eval_jac(self, x, out=None):
        return self._eval_vec(self.lib.gn_eval_jac, x, self.sizes.jac_nnz, out=out)

    def eval_fg(self, x, g_out=None):
        """Line-search trial point: (ok, f, g) from one call, no derivative work."""
        g_out = np.empty(self.n_cons()) if g_out is None else g_out
        f = np.empty(1)
        err = GnError()
        ok = self._record(self.lib.gn_eval_fg(self.h, _f64(x), _f64(f), _f64(g_out), GN_MEM_HOST,
                                              C.byref(err)), err)
        return ok, float(f[0]), g_out

    def eval_hess(self, x, row_weights, obj_weight: float, out=None):
        out = np.empty(self.sizes.hess_nnz) if out is None else out
        err = GnError()
        ok = self._record(self.lib.gn_eval_hess(self.h, _f64(x), _f64(row_weights),
                                                float(obj_weight), _f64(out), GN_MEM_HOST,
                                                C.byref(err)), err)
        return ok, out

    def eval_all(self, x, row_weights, obj_weight: float, outs=None, mem: int = GN_MEM_HOST):
        """f, grad, g, J, H in one call / one launch (gn_eval_all).  outs = (f[1], grad, g,
        jac, hess) host arrays or device tensors; returns (ok, outs)."""
        s = self.sizes
        if outs is None:
            outs = (np.zeros(1), np.empty(s.n_vars), np.empty(s.n_cons), np.empty(s.jac_nnz),
                    np.empty(s.hess_nnz))
        err = GnError()
        ok = self._record(self.lib.gn_eval_all(self.h, _f64(x), _f64(row_weights),
                                               float(obj_weight), *map(_f64, outs), mem,
                                               C.byref(err)), err)
        return ok, outs

    # ---- device-resident variants (pointers to device memory)
    def eval_device(self, which: str, x, out, w=None, ow: float = 1.0, sync: bool = True):
        mem = GN_MEM_DEVICE if sync else GN_MEM_DEVICE_ASYNC
        err = GnError()
        L = self.lib
        if which == "f":
            rc = L.gn_eval_f(self.h, _f64(x), _f64(out), mem, C.byref(err))
        elif which == "grad":
            rc = L.gn_eval_grad(self.h, _f64(x), _f64(out), mem, C.byref(err))
        elif which == "g":
            rc = L.gn_eval_g(self.h, _f64(x), _f64(out), mem, C.byref(err))
        elif which == "jac":
            rc = L.gn_eval_jac(self.h, _f64(x), _f64(out), mem, C.byref(err))
        elif which == "fg":  # out = (f, g) device buffers
            rc = L.gn_eval_fg(self.h, _f64(x), _f64(out[0]), _f64(out[1]), mem, C.byref(err))
        elif which == "hess":
            rc = L.gn_eval_hess(self.h, _f64(x), _f64(w), float(ow), _f64(out), mem,
                                C.byref(err))
        else:
            raise ValueError(which)
        return self._record(rc, err)

    def shard_info(self) -> dict:
        info = (C.c_int64 * 12)()
        gens = np.zeros(max(self.net.n_gen, 1), np.int32)
        _check(self.lib.gn_ctx_shard_info(self.h, info, _i32(gens)))
        keys = ("t0", "T_total", "prev", "next", "n_ramp_gens", "n_base", "ghost_prev0",
                "ghost_next0", "ramp_row0", "ramp_rows_per_gen", "first_step", "owned_lifted")
        d = dict(zip(keys, list(info)))
        d["ramp_gens"] = gens[: d["n_ramp_gens"]].copy()
        return d

    def status(self):
        err = GnError()
        return self._record(self.lib.gn_ctx_status(self.h, C.byref(err)), err)

    def set_stream(self, stream_handle: int):
        """Launch on the caller's stream.  torch's default stream has handle 0, which
        the C-ABI reads as "reset"; it is passed as cudaStreamLegacy instead, so the
        work stays ordered with the caller's default-stream kernels."""
        _check(self.lib.gn_ctx_set_stream(self.h, C.c_void_p(_stream_arg(stream_handle))))

    def reset_stream(self):
        """Back to the context's own (non-blocking) stream."""
        _check(self.lib.gn_ctx_set_stream(self.h, None))

    # ---- lifted problem (lifted.hpp:25-100)
    def lift(self, relax: float):
        err = GnError()
        _check(self.lib.gn_lifted_create(self.h, relax, C.byref(err)), err, "gn_lifted_create")
        self._sizes()
        return self

    def lifted_structure(self):
        s = self.sizes
        n, m = s.n_free, s.n_cons
        nj, nh = s.jac_nnz_lifted, s.hess_nnz_lifted
        f2f = np.empty(n, np.int32)
        jr, jc, jp = (np.empty(nj, np.int32) for _ in range(3))
        hr, hc, hp = (np.empty(nh, np.int32) for _ in range(3))
        sl, su = np.empty(m), np.empty(m)
        _check(self.lib.gn_lifted_structure(self.h, _i32(f2f), _i32(jr), _i32(jc), _i32(jp),
                                            _i32(hr), _i32(hc), _i32(hp), _f64(sl), _f64(su),
                                            GN_MEM_HOST))
        return dict(free_to_full=f2f, jac_rows=jr, jac_cols=jc, jac_pick=jp, hess_rows=hr,
                    hess_cols=hc, hess_pick=hp, s_lower=sl, s_upper=su)


    def publish(self, on: bool = True):
        """gn_ctx_publish: a CondensedKkt later built from this problem's lifted COO arrays
        (as the reference IpmSolver builds it) is recognised and gets the OPF kernels."""
        _check(self.lib.gn_ctx_publish(self.h, 1 if on else 0))
        self._sizes()

    def lifted_gather(self, which: str, full, out=None, mem: int = GN_MEM_HOST):
        """LiftedProblem's value gather (lifted.hpp:144-159): full J (which="jac") or H
        ("hess") values -> lifted values, through host arrays or device tensors."""
        s = self.sizes
        k = s.jac_nnz_lifted if which == "jac" else s.hess_nnz_lifted
        if out is None:
            out = np.empty(k)
        fn = self.lib.gn_lifted_gather_jac if which == "jac" else self.lib.gn_lifted_gather_hess
        _check(fn(self.h, _f64(full), _f64(out), mem))
        return out

    def lifted_eval(self, which: str, x_free, w=None, ow: float = 1.0, out=None,
                    mem: int = GN_MEM_HOST):
        """LiftedProblem::eval_* (lifted.hpp:128-159) on the device: x_free [n_free] ->
        f, grad [n_free], g [m], jac / hess lifted values; "fg" returns (f, g).  Returns
        (ok, out) like the full-space calls (evaluation failures -> ok False)."""
        s = self.sizes
        L = self.lib
        err = GnError()
        size = {"f": 1, "grad": s.n_free, "g": s.n_cons, "jac": s.jac_nnz_lifted,
                "hess": s.hess_nnz_lifted, "fg": s.n_cons}[which]
        if out is None:
            out = np.empty(size)
        if which == "hess":
            rc = L.gn_lifted_eval_hess(self.h, _f64(x_free), _f64(w), float(ow), _f64(out), mem,
                                       C.byref(err))
        elif which == "fg":
            f = np.empty(1) if mem == GN_MEM_HOST else out[1]
            g = out if mem == GN_MEM_HOST else out[0]
            rc = L.gn_lifted_eval_fg(self.h, _f64(x_free), _f64(f), _f64(g), mem, C.byref(err))
            ok = self._record(rc, err)
            return ok, ((float(f[0]), g) if mem == GN_MEM_HOST else out)
        else:
            fn = getattr(L, f"gn_lifted_eval_{which}")
            rc = fn(self.h, _f64(x_free), _f64(out), mem, C.byref(err))
        return self._record(rc, err), out


class CondensedKkt:
    """ipm::CondensedKkt structure + set_jacobian + assemble on the device."""

    def __init__(self, n=None, m=None, jac_rows=None, jac_cols=None, hess_rows=None,
                 hess_cols=None, device: int = 0, nlp: OpfNlp | None = None):
        self.lib = abi.lib()
        h = C.c_void_p()
        err = GnError()
        if nlp is not None:
            rc = self.lib.gn_kkt_create_lifted(nlp.h, C.byref(h), C.byref(err))
            self._nlp = nlp
        else:
            jr = np.ascontiguousarray(jac_rows, np.int32)
            jc = np.ascontiguousarray(jac_cols, np.int32)
            hr = np.ascontiguousarray(hess_rows, np.int32)
            hc = np.ascontiguousarray(hess_cols, np.int32)
            rc = self.lib.gn_kkt_create(n, m, len(jr), _i32(jr), _i32(jc), len(hr), _i32(hr),
                                        _i32(hc), device, C.byref(h), C.byref(err))
        _check(rc, err, "gn_kkt_create")
        self.h = h
        d = (C.c_int64 * 9)()
        self.lib.gn_kkt_dims(h, d)
        self.dim, self.a_nnz, self.m_nnz, self.pair_count, self.jac_nnz, self.hess_nnz, \
            self.n_rows, self.opf_ready, self.fused_ready = list(d)

    def close(self):
        if getattr(self, "h", None):
            self.lib.gn_kkt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def structure(self):
        rp = np.empty(self.n_rows + 1, np.int32)
        ci = np.empty(self.a_nnz, np.int32)
        cp = np.empty(self.dim + 1, np.int32)
        ri = np.empty(self.m_nnz, np.int32)
        _check(self.lib.gn_kkt_structure(self.h, _i32(rp), _i32(ci), _i32(cp), _i32(ri),
                                         GN_MEM_HOST))
        return rp, ci, cp, ri

    def slots(self):
        js = np.empty(self.jac_nnz, np.int32)
        hs = np.empty(self.hess_nnz, np.int32)
        ps = np.empty(self.pair_count, np.int32)
        ds = np.empty(self.dim, np.int32)
        _check(self.lib.gn_kkt_slots(self.h, _i32(js), _i32(hs), _i32(ps), _i32(ds),
                                     GN_MEM_HOST))
        return js, hs, ps, ds

    def set_stream(self, stream_handle: int):
        """As OpfNlp.set_stream (handle 0 = the legacy default stream)."""
        _check(self.lib.gn_kkt_set_stream(self.h, C.c_void_p(_stream_arg(stream_handle))))

    def reset_stream(self):
        """Back to the KKT's own stream (its context's for a lifted KKT)."""
        _check(self.lib.gn_kkt_set_stream(self.h, None))

    def set_grid_cap(self, ctas_per_sm: int):
        """Resident CTAs per SM for the KKT kernels (0 = uncapped)."""
        _check(self.lib.gn_kkt_set_grid_cap(self.h, int(ctas_per_sm)))

    def set_algorithm(self, algo: int):
        _check(self.lib.gn_kkt_set_algorithm(self.h, algo))

    def set_jacobian(self, jvals, mem: int = GN_MEM_HOST):
        _check(self.lib.gn_kkt_set_jacobian(self.h, _f64(jvals), mem))

    def assemble(self, hvals, sigma_x, sigma_s, delta_w: float, delta_c: float,
                 mem: int = GN_MEM_HOST):
        _check(self.lib.gn_kkt_assemble(self.h, _f64(hvals), _f64(sigma_x), _f64(sigma_s),
                                        float(delta_w), float(delta_c), mem))

    def set_jacobian_x(self, x, mem: int = GN_MEM_HOST):
        """A = set_jacobian(eval_jac(x)) computed from x (fused path)."""
        _check(self.lib.gn_kkt_set_jacobian_x(self.h, _f64(x), mem))

    def assemble_x(self, x, row_weights, obj_weight, sigma_x, sigma_s, delta_w, delta_c,
                   mem: int = GN_MEM_HOST):
        """M = assemble(eval_hess(x, w, ow), ...) computed from x (fused path)."""
        _check(self.lib.gn_kkt_assemble_x(self.h, _f64(x), _f64(row_weights), float(obj_weight),
                                          _f64(sigma_x), _f64(sigma_s), float(delta_w),
                                          float(delta_c), mem))

    def update_x(self, x, row_weights, obj_weight, sigma_x, sigma_s, delta_w, delta_c,
                 mem: int = GN_MEM_HOST):
        """set_jacobian_x + assemble_x at the same x in one call (gn_kkt_update_x)."""
        _check(self.lib.gn_kkt_update_x(self.h, _f64(x), _f64(row_weights), float(obj_weight),
                                        _f64(sigma_x), _f64(sigma_s), float(delta_w),
                                        float(delta_c), mem))

    def values(self, a=None, m=None):
        a = np.empty(self.a_nnz) if a is None else a
        m = np.empty(self.m_nnz) if m is None else m
        _check(self.lib.gn_kkt_values(self.h, _f64(a), _f64(m), GN_MEM_HOST))
        return a, m

    def values_ptr(self):
        """Device addresses (ints) of the KKT's own A and M value arrays (gn_kkt_values_ptr)."""
        a, m = C.c_void_p(), C.c_void_p()
        _check(self.lib.gn_kkt_values_ptr(self.h, C.byref(a), C.byref(m)))
        return a.value or 0, m.value or 0

    def values_start(self, a_out=None, m_out=None):
        """gn_kkt_values_start: A / M into pinned host buffers on a side stream (async)."""
        _check(self.lib.gn_kkt_values_start(self.h, _f64(a_out) if a_out is not None else None,
                                            _f64(m_out) if m_out is not None else None))

    def values_wait(self):
        _check(self.lib.gn_kkt_values_wait(self.h))

    def values_device(self, a_out, m_out, sync: bool = True):
        _check(self.lib.gn_kkt_values(self.h, _f64(a_out), _f64(m_out),
                                      GN_MEM_DEVICE if sync else GN_MEM_DEVICE_ASYNC))


def compress_to_csc(nrows, ncols, rows, cols):
    rows = np.ascontiguousarray(rows, np.int32)
    cols = np.ascontiguousarray(cols, np.int32)
    nnz = len(rows)
    cp = np.empty(ncols + 1, np.int32)
    ri = np.empty(max(nnz, 1), np.int32)
    sm = np.empty(max(nnz, 1), np.int32)
    out = C.c_int32()
    err = GnError()
    _check(abi.lib().gn_compress_to_csc(nrows, ncols, nnz, _i32(rows), _i32(cols), _i32(cp),
                                        _i32(ri), _i32(sm), C.byref(out), C.byref(err)), err,
           "compress_to_csc")
    return cp, ri[: out.value], sm[:nnz]


__all__ = ["OpfNlp", "CondensedKkt", "GridError", "load_profile", "compress_to_csc",
           "GN_MEM_HOST", "GN_MEM_DEVICE", "GN_MEM_DEVICE_ASYNC", "GN_IN_FULL"]


class Ipm:
    """Device-resident IPM vector operations (gn_ipm_*) on the lifted
    problem of `kkt` (a CondensedKkt(nlp=...)).  Vectors are CUDA tensors (float64);
    iterates / residuals / directions are sequences in the field order
    x s y zlx zux zls zus.  Scalars come back as Python floats unless `sync=False`."""

    def __init__(self, kkt: CondensedKkt, x_lower, x_upper, s_lower, s_upper):
        import torch
        self.lib = abi.lib()
        self.kkt = kkt
        dev = torch.device("cuda", torch.cuda.current_device())
        t = lambda a: (a if hasattr(a, "data_ptr") else  # noqa: E731
                       torch.from_numpy(np.ascontiguousarray(a, np.float64))).to(dev)
        self._b = [t(x_lower), t(x_upper), t(s_lower), t(s_upper)]
        h = C.c_void_p()
        err = GnError()
        _check(self.lib.gn_ipm_create(kkt.h, *[b.data_ptr() for b in self._b], GN_MEM_DEVICE,
                                      C.byref(h), C.byref(err)), err, "gn_ipm_create")
        self.h = h
        self._out = torch.zeros(4, dtype=torch.float64, device=dev)

    def close(self):
        if getattr(self, "h", None):
            self.lib.gn_ipm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _s(cls, arrays):
        return cls(*[a.data_ptr() if a is not None else None for a in arrays])

    def _mem(self, sync):
        return GN_MEM_DEVICE if sync else GN_MEM_DEVICE_ASYNC

    def _scalar(self, k, sync):
        return [float(v) for v in self._out[:k].cpu()] if sync else self._out[:k]

    def jac_transpose_multiply(self, jv, y, out, sync=True):
        _check(self.lib.gn_ipm_jac_transpose_multiply(self.h, jv.data_ptr(), y.data_ptr(),
                                                      out.data_ptr(), self._mem(sync)))

    def jac_multiply(self, jv, x, out, sync=True):
        _check(self.lib.gn_ipm_jac_multiply(self.h, jv.data_ptr(), x.data_ptr(), out.data_ptr(),
                                            self._mem(sync)))

    def residuals(self, it, grad, g, jv, mu, r, sync=True):
        _check(self.lib.gn_ipm_residuals(self.h, C.byref(self._s(abi.GnIterate, it)),
                                         grad.data_ptr(), g.data_ptr(), jv.data_ptr(), mu,
                                         C.byref(self._s(abi.GnResiduals, r)), self._mem(sync)))

    def bound_condensation(self, it, r, sx, ss, qx, qs, sync=True):
        _check(self.lib.gn_ipm_bound_condensation(
            self.h, C.byref(self._s(abi.GnIterate, it)), C.byref(self._s(abi.GnResiduals, r)),
            sx.data_ptr(), ss.data_ptr(), qx.data_ptr(), qs.data_ptr(), self._mem(sync)))

    def fraction_to_boundary(self, it, d, tau, sync=True):
        _check(self.lib.gn_ipm_fraction_to_boundary(
            self.h, C.byref(self._s(abi.GnIterate, it)), C.byref(self._s(abi.GnDirection, d)),
            tau, self._out.data_ptr(), self._mem(sync)))
        return self._scalar(2, sync)

    def barrier_value(self, f, x, s, mu, sync=True):
        _check(self.lib.gn_ipm_barrier_value(self.h, f, x.data_ptr(), s.data_ptr(), mu,
                                             self._out.data_ptr(), self._mem(sync)))
        return self._scalar(1, sync)

    def barrier_slope(self, grad, it, d, mu, sync=True):
        _check(self.lib.gn_ipm_barrier_slope(
            self.h, grad.data_ptr(), C.byref(self._s(abi.GnIterate, it)),
            C.byref(self._s(abi.GnDirection, d)), mu, self._out.data_ptr(), self._mem(sync)))
        return self._scalar(1, sync)

    def constraint_violation(self, g, s, sync=True):
        _check(self.lib.gn_ipm_constraint_violation(self.h, g.data_ptr(), s.data_ptr(),
                                                    self._out.data_ptr(), self._mem(sync)))
        return self._scalar(1, sync)

    def kkt_error(self, it, r, mu, sync=True):
        _check(self.lib.gn_ipm_kkt_error(self.h, C.byref(self._s(abi.GnIterate, it)),
                                         C.byref(self._s(abi.GnResiduals, r)), mu,
                                         self._out.data_ptr(), self._mem(sync)))
        return self._scalar(3, sync)

    def recover_bound_steps(self, it, r, d, sync=True):
        _check(self.lib.gn_ipm_recover_bound_steps(
            self.h, C.byref(self._s(abi.GnIterate, it)), C.byref(self._s(abi.GnResiduals, r)),
            C.byref(self._s(abi.GnDirection, d)), self._mem(sync)))

    def solve_rhs(self, qx, qs, qy, ss, dw, dc, rhs, sync=True):
        _check(self.lib.gn_kkt_solve_rhs(self.h, qx.data_ptr(), qs.data_ptr(), qy.data_ptr(),
                                         ss.data_ptr(), dw, dc, rhs.data_ptr(), self._mem(sync)))

    def solve_finish(self, dx, qs, qy, ss, dw, dc, ds, dy, sync=True):
        _check(self.lib.gn_kkt_solve_finish(self.h, dx.data_ptr(), qs.data_ptr(), qy.data_ptr(),
                                            ss.data_ptr(), dw, dc, ds.data_ptr(), dy.data_ptr(),
                                            self._mem(sync)))
