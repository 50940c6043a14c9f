"""One launch each of the §8(f) kernels at bench sizes, for an ncu capture
(scripts/gpu_ncu_frows.sh): bq_binary_op AND on 256 MiB operands, the K7 encoder on
a 2^22-word C2 bitmap, and the NVRTC SSum(64, 32) program over the C2 inputs."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_4073_b200 as bq  # noqa: E402
from paper_1402_4073_b200 import _lib, api  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
n, nw = 64, 1 << 22
qs = np.asarray([lib.bq_gen_density_q16(1402, i, 655, 32768) for i in range(n)], dtype=np.uint32)
data = torch.empty((n, nw), dtype=torch.int64, device=dev)
_lib.check(lib.bq_gen_bernoulli_rows(1402, 0, n, qs.ctypes.data, 0, nw, data.data_ptr(), nw, s))
pc = torch.zeros(1, dtype=torch.int64, device=dev)
lnz = torch.zeros(1, dtype=torch.int64, device=dev)
big_a, big_b = data[0:8].reshape(-1), data[8:16].reshape(-1)
out = torch.empty(8 * nw, dtype=torch.int64, device=dev)
mixed = data[20]
enc = torch.empty(nw + 2, dtype=torch.int64, device=dev)
q = bq.ThresholdQuery([data[i] for i in range(n)], 64 * nw)
prog = api.compile_program(api.CircuitLibrary(64, "sideways").program(64, 32))
for rep in range(2):
    _lib.check(lib.bq_binary_op(0, big_a.data_ptr(), 8 * nw, big_b.data_ptr(), 8 * nw, 64 * 8 * nw, out.data_ptr(),
                                pc.data_ptr(), lnz.data_ptr(), s))
    k = ctypes.c_uint64(0)
    _lib.check(lib.bq_rle_encode_device(mixed.data_ptr(), nw, 64 * nw, enc.data_ptr(), nw + 2, ctypes.byref(k), s))
    prog.run(q, out, pc, lnz)
    torch.cuda.synchronize()
print("ok")
