"""C4 streams, K4s time per query across thresholds (phase C grows as T falls).

L2 flushed (256 MB) before each timed launch, as bench.py does."""
import ctypes
import json
import statistics
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1402_4073_b200 as bq  # noqa: E402

lib = bq._lib.load()
n, r = 1024, 1 << 30


def markov(i):
    cap = (r // 64) // 8 + 4096
    while True:
        buf = np.empty(cap, dtype=np.uint64)
        k = ctypes.c_uint64(0)
        if lib.bq_gen_markov_rle(1402, i, r, 256.0, 12544.0, buf.ctypes.data, cap, ctypes.byref(k)) == 0:
            return buf[: k.value].copy()
        cap *= 2


with ThreadPoolExecutor(16) as ex:
    streams = list(ex.map(markov, range(n)))
d = [torch.from_numpy(s.view(np.int64)).cuda() for s in streams]
q = bq.RleQuery(d, r)
out = torch.empty(r // 64, dtype=torch.int64, device="cuda")
pc = torch.zeros(1, dtype=torch.int64, device="cuda")
q.threshold(50, out, pc)
q.threshold(50, out, pc)
res = {}
scratch = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
TS = [int(x) for x in sys.argv[1:]] or [1, 2, 5, 10, 20, 30, 50, 100, 1024]
cases = [(f"T={t}", (lambda t=t: q.threshold(t, out, pc))) for t in TS]
if len(sys.argv) == 1:
    cases.append(("interval[3,40]", lambda: q.symmetric([3 <= k <= 40 for k in range(n + 1)], out, pc)))
for label, fn in cases:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev:
        scratch.add_(1)  # L2 flush; also gives the host time to queue the query (kernel time only)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    pc.zero_()
    fn()
    res[label] = {"ms": round(statistics.median(a.elapsed_time(b) for a, b in ev), 4), "popcount": int(pc.item())}
print(json.dumps(res))
