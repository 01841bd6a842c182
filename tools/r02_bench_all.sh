#!/bin/bash
# Round-2 bench sweep on one B200 (run under gpurun): every config's default line,
# the general (unguarded) kernels' lines, the reference arm, the int8 library peak.
T=${1:-r02e}
python tools/int8_peak.py > gpurun_out/${T}_int8_peak.log 2>&1
for c in 4 2 3 5; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_c$c.json 2> gpurun_out/${T}_bench_c$c.err
  echo "c$c rc=$?"
done
for c in 2 3 5; do
  python bench.py --config $c --steps 3 --warmup 1 --no-fastpath --no-opt-in --no-e2e --no-cpu-baseline \
    > gpurun_out/${T}_bench_c${c}_general.json 2> gpurun_out/${T}_bench_c${c}_general.err
  echo "c$c general rc=$?"
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref_c4.json 2> gpurun_out/${T}_ref_c4.err
echo "ref rc=$?"
nproc > gpurun_out/${T}_nproc.txt; lscpu > gpurun_out/${T}_lscpu.txt
