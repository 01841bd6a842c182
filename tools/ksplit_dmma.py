"""Split-k on the DMMA path at one size: every schedule x forced split depth, with the
cluster/DSMEM merge (default) and with the global-memory protocols
(STARMM_DMMA_CLUSTER=0).  Device time of 20 back-to-back asynchronous executes per
point (CUDA events), fp64 N(0,1) inputs.  Prints one JSON object.

  python tools/ksplit_dmma.py [n] [algos]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_05328_b200 as sm  # noqa: E402
from paper_1911_05328_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
algos = sys.argv[2].split(",") if len(sys.argv) > 2 else ["co2", "co3", "tar", "sar", "star"]
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
B = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
res = {"n": n}
for cluster in ("1", "0"):
    os.environ["STARMM_DMMA_CLUSTER"] = cluster
    for algo in algos:
        for ks in ((-1,) if algo == "co2" else (-1, 0, 1, 2, 3)):
            p = _lib.Plan(_lib.SR_FP64, algo, "pooled", n, n, n, 64, 148, ks, 0, _lib.F_ASYNC)
            run = lambda: p.execute(C.data_ptr(), n, A.data_ptr(), n, B.data_ptr(), n, stream)  # noqa: E731
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            st = p.stats()
            res[f"{algo}_ks{ks}_cl{cluster}"] = {"ms": round(ms, 4), "tops": round(2 * n ** 3 / ms / 1e9, 2),
                                                 "S": st["ksplit"], "cluster": st["cluster_size"]}
            p.close()
print(json.dumps(res))
