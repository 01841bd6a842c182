nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/sweep tools/sweep_dmma.cu || exit 1
/tmp/sweep 16384 > gpurun_out/sweep_group.jsonl || exit 1
for g in 4 8 24 64; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:dmma -s 1 -c 1 --csv /tmp/sweep 16384 $g 2>/dev/null | grep -E "dram__bytes_read|hit_rate|duration" | sed "s/^/g=$g,/" >> gpurun_out/ncu_group.csv
done
echo ok
