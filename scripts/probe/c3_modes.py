"""C3 shape (N=256, 2 GiB): K2 time per epilogue mode (BREAK with few / many breakpoints, LUT, parity)."""
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1402_4073_b200 as bq  # noqa: E402

lib = bq._lib.load()
n, nw = 256, 1 << 20
data = torch.empty((n, nw), dtype=torch.int64, device="cuda")
q16 = np.full(n, 3277, dtype=np.uint32)
assert lib.bq_gen_bernoulli_rows(1402, 0, n, q16.ctypes.data, 0, nw, data.data_ptr(), nw,
                                 torch.cuda.current_stream().cuda_stream) == 0
q = bq.ThresholdQuery([data[i] for i in range(n)], 64 * nw)
rng = np.random.default_rng(1)
specs = {
    "interval[2,10]": [2 <= k <= 10 for k in range(n + 1)],
    "threshold 13": [k >= 13 for k in range(n + 1)],
    "parity": [k % 2 == 1 for k in range(n + 1)],
    "mod4==1": [k % 4 == 1 for k in range(n + 1)],
    "20 breakpoints": [bool((k // 3) % 2) if k < 60 else False for k in range(n + 1)],
    "random (LUT)": [bool(x) for x in rng.integers(0, 2, n + 1)],
}
out = torch.empty(nw, dtype=torch.int64, device="cuda")
pc = torch.zeros(1, dtype=torch.int64, device="cuda")
res = {}
for name, acc in specs.items():
    for _ in range(3):
        q.symmetric(acc, out, pc)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev:
        a.record()
        q.symmetric(acc, out, pc)
        b.record()
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    res[name] = {"ms": round(ms, 4), "GB/s": round(n * nw * 8 / (ms / 1e3) / 1e9, 1)}
print(json.dumps(res))
