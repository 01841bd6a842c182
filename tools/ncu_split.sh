#!/bin/bash
# ncu --set full of the round-2 split-k kernels at n = 2048 fp64 (one GPU):
#   cluster: sar S=2 on thread-block clusters (DSMEM merge); balanced: tar auto (stream-K)
T=${1:-r02n}
python tools/one_mm.py float sar 2048 1 2 || exit 1
ncu --set full --clock-control none --import-source on -k regex:cluster -s 1 -c 1 \
    -o gpurun_out/${T}_prof_cluster python tools/one_mm.py float sar 2048 1 2 > gpurun_out/${T}_ncu_cluster.log 2>&1
ncu -i gpurun_out/${T}_prof_cluster.ncu-rep --page raw --csv > gpurun_out/${T}_prof_cluster.raw.csv 2>/dev/null
ncu -i gpurun_out/${T}_prof_cluster.ncu-rep --page details --csv > gpurun_out/${T}_prof_cluster.details.csv 2>/dev/null
python tools/one_mm.py float tar 2048 -1 2 || exit 2
ncu --set full --clock-control none --import-source on -k regex:balanced -s 1 -c 1 \
    -o gpurun_out/${T}_prof_balanced python tools/one_mm.py float tar 2048 -1 2 > gpurun_out/${T}_ncu_balanced.log 2>&1
ncu -i gpurun_out/${T}_prof_balanced.ncu-rep --page raw --csv > gpurun_out/${T}_prof_balanced.raw.csv 2>/dev/null
ncu -i gpurun_out/${T}_prof_balanced.ncu-rep --page details --csv > gpurun_out/${T}_prof_balanced.details.csv 2>/dev/null
rm -f gpurun_out/${T}_prof_*.ncu-rep
echo done
