#!/bin/bash
# round-2 validation on one B200: GPU suite, smoke, the driver's default bench and
# reference arm, and every config's bench line.
T=${1:-r02t}
python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|^FAILED" gpurun_out/${T}_pytest.log | tail -5
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref_default.json 2> gpurun_out/${T}_ref_default.err; echo "ref rc=$?"
for c in 2 3 5; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_c$c.json 2> gpurun_out/${T}_bench_c$c.err; echo "c$c rc=$?"
done
# the reference's own leaf kernel, single thread, on this box's host
python tools/ref_cpu_sweep.py --native-matmul > gpurun_out/${T}_native_matmul.log 2>&1 && cp profiles/r02_ref_native_matmul.json gpurun_out/; echo "native rc=$?"
# launch list of the default bench command (ncu, serialised, cold cache: shares only)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_default.csv \
    python bench.py --gpus 1 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/${T}_gpu.txt
