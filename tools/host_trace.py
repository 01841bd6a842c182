"""Timeline of the host-buffer schedule (starmm_execute_host, STARMM_HOST_TRACE=1).

  python tools/host_trace.py <config 2|3|4|5> [n]      -> gpurun_out/host_trace_c<cfg>.txt

Runs Executor.execute_host twice on pinned buffers shaped like the bench's config
(the second run is traced) and prints the wall time; the per-event lines go to stderr."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_05328_b200 as sm  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) else {2: 4096, 3: 8192, 4: 16384, 5: 16384}[cfg]
br = int(sys.argv[3]) if len(sys.argv) > 3 else 0       # phase-2 block rows (0 = auto)
g = torch.Generator().manual_seed(cfg)
if cfg == 4:
    s = sm.FLOAT_RING
    A = torch.randn(n, n, dtype=torch.float64, generator=g)
    B = torch.randn(n, n, dtype=torch.float64, generator=g)
    C = torch.rand(n, n, dtype=torch.float64, generator=g) * 2 - 1
elif cfg == 2:
    s = sm.INT_RING
    A = torch.randint(-16, 17, (n, n), dtype=torch.int64, generator=g)
    B = torch.randint(-16, 17, (n, n), dtype=torch.int64, generator=g)
    C = torch.zeros(n, n, dtype=torch.int64)
else:
    s = sm.TROPICAL_F32 if cfg == 3 else sm.TROPICAL_I32
    dt = torch.float32 if cfg == 3 else torch.int32
    if cfg == 3:
        W = torch.randint(1, 101, (n, n), generator=g).to(dt)
        W[torch.rand(n, n, generator=g) >= 0.1] = float("inf")
    else:
        W = torch.randint(1, 10 ** 6 + 1, (n, n), generator=g, dtype=dt)
    W.fill_diagonal_(0)
    A = B = W
    C = W.clone()
A = A.pin_memory()
B = A if B is not None and B.data_ptr() == A.data_ptr() else B.pin_memory()
C = C.pin_memory()
C0 = C.clone()
with sm.Executor(sm.Config(base_dim=64, workers=148, allow_nonpow2=True)) as ex:
    ex.execute_host("star", C, A, B, s, block_rows=br)
    torch.cuda.synchronize()
    C.copy_(C0)
    os.environ["STARMM_HOST_TRACE"] = "1"
    t0 = time.perf_counter()
    ex.execute_host("star", C, A, B, s, block_rows=br)
    t = time.perf_counter() - t0
    del os.environ["STARMM_HOST_TRACE"]
    ts = []
    for _ in range(3):
        C.copy_(C0)
        t1 = time.perf_counter()
        ex.execute_host("star", C, A, B, s, block_rows=br)
        ts.append(time.perf_counter() - t1)
print(f"config {cfg} n={n} block_rows={br} phase1={os.environ.get('STARMM_HOST_PHASE1', '1')} "
      f"ksplit2={os.environ.get('STARMM_HOST_KSPLIT2', 'auto')}: traced {t * 1e3:.2f} ms; untraced {min(ts) * 1e3:.2f} ms "
      f"= {2 * n ** 3 / min(ts) / 1e12:.2f} Tops/s e2e; executes {ex.last_stats['executes']}")
