set -x
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain4.log 2>&1 && \
$B --config 3 > gpurun_out/plain3.log 2>&1 && \
$B --config 5 --n 16384 > gpurun_out/plain5.log 2>&1 && \
$B --config 2 > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_l4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dmma -c 1 -o gpurun_out/prof_c4_dmma $B > gpurun_out/ncu_f4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:simt_mm -c 1 -o gpurun_out/prof_c3_simt $B --config 3 > gpurun_out/ncu_f3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:simt_mm -c 1 -o gpurun_out/prof_c5_simt $B --config 5 --n 16384 > gpurun_out/ncu_f5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:simt_mm -c 1 -o gpurun_out/prof_c2_simt $B --config 2 > gpurun_out/ncu_f2.log 2>&1
echo rc=$?
