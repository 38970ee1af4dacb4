import sys, faulthandler
faulthandler.enable()
import torch
print('torch', torch.cuda.is_available(), flush=True)
import numpy as np
from paper_2405_14032_b200.network import synthetic_case
from paper_2405_14032_b200.opf import OpfNlp, CondensedKkt, load_profile
from paper_2405_14032_b200.abi import GN_MEM_DEVICE_ASYNC as A
raw = synthetic_case(300, 470, 60, 250, seed=3); net = raw.network(); T = 24
print('net', flush=True)
nlp = OpfNlp(net, T, load_profile(net.n_load, T)); nlp.lift(1e-4); K = CondensedKkt(nlp=nlp)
print('kkt', flush=True)
s = nlp.sizes; dev = torch.device("cuda")
xl, xu, xs, _, _ = nlp.bounds()
dx = torch.tensor(xs, device=dev); dw = torch.ones(s.n_cons, dtype=torch.float64, device=dev)
dsx = torch.ones(s.n_free, dtype=torch.float64, device=dev); dss = torch.ones(s.n_cons, dtype=torch.float64, device=dev)
f = torch.zeros(1, dtype=torch.float64, device=dev); g = torch.zeros(s.n_cons, dtype=torch.float64, device=dev)
gr = torch.zeros(s.n_vars, dtype=torch.float64, device=dev); J = torch.zeros(s.jac_nnz, dtype=torch.float64, device=dev)
H = torch.zeros(s.hess_nnz, dtype=torch.float64, device=dev)
st = torch.cuda.Stream(); nlp.set_stream(st.cuda_stream); K.set_stream(st.cuda_stream)
calls = {
 "f": lambda: nlp.eval_device("f", dx, f, sync=False),
 "grad": lambda: nlp.eval_device("grad", dx, gr, sync=False),
 "g": lambda: nlp.eval_device("g", dx, g, sync=False),
 "jac": lambda: nlp.eval_device("jac", dx, J, sync=False),
 "hess": lambda: nlp.eval_device("hess", dx, H, w=dw, ow=1.0, sync=False),
 "setjx": lambda: K.set_jacobian_x(dx, mem=A),
 "asmx": lambda: K.assemble_x(dx, dw, 1.0, dsx, dss, 1e-4, 1e-8, mem=A),
}
print('eager', flush=True)
for k, fn in calls.items():
    print(' call', k, flush=True)
    with torch.cuda.stream(st):
        fn()
    torch.cuda.synchronize()
print('capture', flush=True)
for k, fn in calls.items():
    print(' cap', k, flush=True)
    g_ = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g_, stream=st):
            fn()
        g_.replay(); torch.cuda.synchronize()
        print(k, "ok")
    except Exception as e:
        print(k, "FAIL", str(e).splitlines()[0])
        torch.cuda.synchronize()
