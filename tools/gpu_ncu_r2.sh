#!/bin/bash
# ncu evidence for round 2 (run under gpurun): the launch list of the bench
# command, per-launch DRAM bytes of one bench step, one full capture of the
# dominant kernel (packed plan as bench.py builds it), and a UFi A/B of the
# dominant layer at matched tile configuration.
TAG=${1:-r2}
CASE=${2:-"512x4608@70%/b128"}
mkdir -p gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-compare --no-cpu --streams 1 > /dev/null 2>&1; echo ncu-launches $?
timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --nvtx --nvtx-include bench_timed/ -k regex:"esc_(rec|spmm)_kernel" -c 90 --csv --log-file gpurun_out/${TAG}_dram.csv python bench.py --steps 1 --warmup 3 --no-compare --no-cpu --streams 1 > /dev/null 2>&1; echo ncu-dram $?
python tools/traffic_from_ncu.py gpurun_out/${TAG}_dram.csv gpurun_out/${TAG}_traffic.json suite "$CASE"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include profile_reps/ -k regex:"esc_(rec|spmm)_kernel" -c 1 -o gpurun_out/${TAG}_full python tools/profile_case.py --case "$CASE" --reps 3 > gpurun_out/${TAG}_full.log 2>&1; echo ncu-full $?
for U in 1 2 3 4; do
  timeout -s KILL 600 ncu --set full --clock-control none --nvtx --nvtx-include profile_reps/ -k regex:"esc_(rec|spmm)_kernel" -c 1 -o gpurun_out/${TAG}_ufi$U python tools/profile_case.py --case "$CASE" --reps 2 --ufi $U > gpurun_out/${TAG}_ufi$U.log 2>&1; echo ncu-ufi$U $?
done
