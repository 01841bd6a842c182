"""General (full-range) int64 (+,x): the CUDA-core kernel (simt_i64) vs the opt-in
radix-256 digit GEMMs on the int8 tensor cores (tcgen05_i8_radix256_int64), same
uniformly random int64 data (every digit populated), device time of 3 asynchronous
executes after 2 warm-ups.  Prints one JSON line per (n, path).
  python tools/int64_general.py [n ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_05328_b200 import _lib  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [4096, 8192, 16384]:
    A = torch.randint(-2 ** 62, 2 ** 62, (n, n), dtype=torch.int64, device="cuda")
    B = torch.randint(-2 ** 62, 2 ** 62, (n, n), dtype=torch.int64, device="cuda")
    C = torch.zeros(n, n, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for flags, name in ((_lib.F_INT_TENSOR | _lib.F_ASYNC, "opt-in tensor"), (_lib.F_ASYNC, "cuda cores")):
        p = _lib.Plan(_lib.SR_INT64, "star", "pooled", n, n, n, 64, 148, -1, 0, flags)
        for _ in range(2):
            p.execute(C.data_ptr(), n, A.data_ptr(), n, B.data_ptr(), n, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            p.execute(C.data_ptr(), n, A.data_ptr(), n, B.data_ptr(), n, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"n": n, "kind": name, "path": p.stats()["path_name"], "ms": round(ms, 3),
                          "tops": round(2 * n ** 3 / ms / 1e9, 2)}))
        p.close()
