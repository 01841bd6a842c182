#!/bin/bash
# ncu evidence for the bench workloads (run under gpurun; one GPU).
# Each profiled command first runs plain and must exit 0 (B200_PROFILING.md).
# usage: bash tools/ncu_capture.sh <tag> [configs...]
#   configs: 2 3 4 5 (default paths), 2t (config 2 --int-tensor), 4e (config 4 --fp64-emu),
#            5f (config 5 at its full n = 49152), 2g / 3g / 5g (the general kernels,
#            --no-fastpath; 5g at n = 16384)
#   launch list : the bench command itself (e2e + cpu baseline legs included)
#   full capture: the tile kernel, from the same command without the e2e / cpu legs
set -x
TAG=${1:-r01}; shift
CFGS=${@:-4 3 5 2}
for c in $CFGS; do
  base=${c:0:1}; X=""; F=""
  [ "$base" = "5" ] && X="--size 16384"
  # the tile kernel by its demangled name (policy included): a plan also launches
  # predicated-off fallback kernels of other policies, which -k regex:simt_mm would catch
  K=simt_mm; [ "$base" = "4" ] && K=dmma_fp64
  [ "$base" = "2" ] && K=PolI8Dp4a; [ "$base" = "3" ] && K=PolS16x2Min; [ "$base" = "5" ] && K=PolF32Pair
  case $c in 2t) F="--int-tensor"; K=tcg_kernel;; 4e) F="--fp64-emu"; K=tcg_kernel;;
             5f) X="";; 2g) F="--no-fastpath"; K="PolI64,";; 3g) F="--no-fastpath"; K=PolF32Pair;; 5g) F="--no-fastpath"; K=PolI32Sat;; esac
  B="python bench.py --steps 2 --warmup 1 --config $base $X $F --no-opt-in"
  $B > gpurun_out/${TAG}_plain_c$c.json 2> gpurun_out/${TAG}_plain_c$c.err || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches_c$c.csv $B > /dev/null 2>&1 || exit 2
  B2="$B --no-e2e --no-cpu-baseline"
  $B2 > /dev/null 2>&1 || exit 3
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$K" -s 1 -c 1 \
      -o gpurun_out/${TAG}_prof_c$c $B2 > gpurun_out/${TAG}_ncu_c$c.log 2>&1 || exit 4
  # raw page as CSV (what tools/summarize_ncu.py reads); the 12-16 MB report only with KEEP_REP=1
  ncu -i gpurun_out/${TAG}_prof_c$c.ncu-rep --page raw --csv > gpurun_out/${TAG}_prof_c$c.raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_prof_c$c.ncu-rep --page details --csv > gpurun_out/${TAG}_prof_c$c.details.csv 2>/dev/null
  [ "$KEEP_REP" = "1" ] || rm -f gpurun_out/${TAG}_prof_c$c.ncu-rep
done
echo done
