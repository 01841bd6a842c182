"""Time one schedule at several forced k-split depths (Config.ksplit) on device inputs."""
import sys, time, json, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_05328_b200 as sm
sid, n = sys.argv[1], int(sys.argv[2])
s = sm.get_semiring(sid)
g = torch.Generator(device="cuda"); g.manual_seed(1)
if sid == "float":
    A = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
elif sid == "int":
    A = torch.randint(-16, 17, (n, n), generator=g, device="cuda", dtype=torch.int64)
    B = torch.randint(-16, 17, (n, n), generator=g, device="cuda", dtype=torch.int64)
else:
    A = torch.randint(1, 101, (n, n), generator=g, device="cuda").to(s.torch_dtype)
    B = torch.randint(1, 101, (n, n), generator=g, device="cuda").to(s.torch_dtype)
res = {}
for algo in (sys.argv[3].split(",") if len(sys.argv) > 3 else ("co2", "star", "tar")):
    for ks in ((None,) if algo == "co2" else (0, 1, 2, 3, None)):
        C = torch.zeros(n, n, dtype=s.torch_dtype, device="cuda")
        with sm.Executor(sm.Config(base_dim=64, workers=148, ksplit=ks)) as ex:
            M, Am, Bm = sm.Matrix(C, s), sm.Matrix(A, s), sm.Matrix(B, s)
            for _ in range(3):
                sm.run_algorithm(ex, algo, M, Am, Bm, s)
            torch.cuda.synchronize(); t = time.perf_counter()
            for _ in range(10):
                sm.run_algorithm(ex, algo, M, Am, Bm, s)
            torch.cuda.synchronize(); t = (time.perf_counter() - t) / 10
            res[f"{algo}_ks{ks}"] = {"ms": round(t * 1e3, 3), "tops": round(2 * n ** 3 / t / 1e12, 1),
                                      "S": ex.last_stats["ksplit"], "path": ex.last_stats["path_name"]}
print(json.dumps(res))
