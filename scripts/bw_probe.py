"""HBM ceilings on this B200 for the roofline discussion: write-only fill,
read-only reduction and copy, over buffers the size of the dominant callback's output
(1.6 GB), CUDA events, best of 10.  Prints one JSON line."""
import json

import torch


def timed(fn, reps=10):
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


def main():
    n = 200 * 1024 * 1024  # 1.68 GB of doubles
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    x.fill_(1.0)
    out = {}
    t = timed(lambda: x.fill_(0.5))
    out["write_only_gbs"] = 8 * n / t / 1e9
    t = timed(lambda: x.sum())
    out["read_only_gbs"] = 8 * n / t / 1e9
    t = timed(lambda: y.copy_(x))
    out["copy_gbs"] = 16 * n / t / 1e9
    out["bytes"] = 8 * n
    print(json.dumps(out))


if __name__ == "__main__":
    main()
