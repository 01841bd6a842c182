#!/bin/bash
# Host-path schedule sweep (run under gpurun): PCIe probe + host_trace variants.
# usage: bash tools/host_sweep.sh <tag> "<cfg>:<block_rows>:<phase1>:<ksplit2>" ...
TAG=$1; shift
timeout 120 python tools/pcie_bw.py > gpurun_out/${TAG}_pcie.json 2>&1
for v in "$@"; do
  IFS=: read c br p1 k2 <<< "$v"
  if [ "$k2" = "auto" ]; then unset STARMM_HOST_KSPLIT2; else export STARMM_HOST_KSPLIT2=$k2; fi
  STARMM_HOST_PHASE1=$p1 timeout 300 python tools/host_trace.py $c 0 $br > gpurun_out/${TAG}_c${c}_b${br}_p${p1}_k${k2}.txt 2>&1
  tail -1 gpurun_out/${TAG}_c${c}_b${br}_p${p1}_k${k2}.txt
done
