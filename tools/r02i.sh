#!/bin/bash
# round-2 batch: new-kernel tests, DMMA split-k A/B, int64 general and config 2 lines
T=r02i
python -m pytest tests/test_gpu_round2.py -q -x > gpurun_out/${T}_round2.log 2>&1; echo "round2 rc=$?"
grep -E "passed|failed|^FAILED|^E " gpurun_out/${T}_round2.log | head -20
python tools/ksplit_dmma.py 2048 > gpurun_out/${T}_ksplit_dmma_2048.json 2> gpurun_out/${T}_ksplit_dmma_2048.err; echo "ks2048 rc=$?"
python tools/ksplit_dmma.py 1024 > gpurun_out/${T}_ksplit_dmma_1024.json 2> gpurun_out/${T}_ksplit_dmma_1024.err; echo "ks1024 rc=$?"
python bench.py --config 2 --steps 3 --warmup 1 --no-fastpath --no-opt-in --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_c2_general.json 2>&1; echo "c2g rc=$?"
python bench.py --config 2 --steps 10 --warmup 3 --no-opt-in --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2>&1; echo "c2 rc=$?"
python bench.py --config 4 --steps 10 --warmup 3 --no-opt-in --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2>&1; echo "c4 rc=$?"
