"""Floor of the C1 timing method: a one-element torch kernel between two CUDA events
after a 256 MB L2 flush (bench.py C1 times each query the same way)."""
import torch, statistics
x = torch.zeros(1, device="cuda"); scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
res = []
for i in range(220):
    scratch.add_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); x.add_(1); b.record(s)
    res.append((a, b))
torch.cuda.synchronize()
t = [a.elapsed_time(b) * 1000 for a, b in res[20:]]
print("tiny kernel between events after L2 flush: median %.2f us, min %.2f us" % (statistics.median(t), min(t)))
