"""Which stream bounds the step at small configurations?  CUDA-graph replay times of the
callbacks alone (one stream), the fused KKT alone (its stream + lanes) and both, as bench.py
runs them.  usage: python scripts/chain_probe.py [config] [periods] [reps]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
from paper_2405_14032_b200.abi import GN_MEM_DEVICE_ASYNC  # noqa: E402
from paper_2405_14032_b200.opf import CondensedKkt, OpfNlp  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "case1354pegase"
periods = int(sys.argv[2]) if len(sys.argv) > 2 else 24
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
raw, net, scale = bench.build_workload(0, 1, periods, config)
dev = torch.device("cuda", 0)
nlp = OpfNlp(net, periods, scale)
cs = torch.cuda.Stream()
ks = torch.cuda.Stream(priority=-1)
nlp.set_stream(cs.cuda_stream)
nlp.lift(1e-4)
kkt = CondensedKkt(nlp=nlp)
kkt.set_grid_cap(2)
kkt.set_stream(ks.cuda_stream)
s = nlp.sizes
xl, xu, xs, _, _ = nlp.bounds()
x, w, sx, ss = bench.inputs((xl, xu, xs), s.n_cons, s.n_free)
f64 = dict(dtype=torch.float64, device=dev)
dx, dw, dsx, dss = (torch.from_numpy(a).to(dev) for a in (x, w, sx, ss))
f = torch.zeros(1, **f64)
grad, g = torch.empty(s.n_vars, **f64), torch.empty(s.n_cons, **f64)
J, H = torch.empty(s.jac_nnz, **f64), torch.empty(s.hess_nnz, **f64)
A = GN_MEM_DEVICE_ASYNC
ev0, ev1 = torch.cuda.Event(), torch.cuda.Event()


def callbacks():  # as the one-GPU bench step: gn_eval_all
    nlp.eval_all(dx, dw, 1.0, outs=(f, grad, g, J, H), mem=A)


def kkt_only():
    ev0.record(cs)
    ks.wait_event(ev0)
    kkt.update_x(dx, dw, 1.0, dsx, dss, 1e-4, 5.6e-9, mem=A)
    ev1.record(ks)
    cs.wait_event(ev1)


def both():
    ev0.record(cs)
    ks.wait_event(ev0)
    kkt.update_x(dx, dw, 1.0, dsx, dss, 1e-4, 5.6e-9, mem=A)
    callbacks()
    ev1.record(ks)
    cs.wait_event(ev1)


out = {"config": config, "periods": periods}
for name, fn in (("callbacks", callbacks), ("kkt", kkt_only), ("both", both)):
    for _ in range(3):
        with torch.cuda.stream(cs):
            fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=cs):
        fn()
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for a, b in evs:
        with torch.cuda.stream(cs):
            a.record(cs)
            gr.replay()
            b.record(cs)
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) for a, b in evs])
    out[name] = {"ms_mean": float(t.mean()), "ms_median": float(np.median(t))}
print(json.dumps(out))
