#!/bin/bash
# One GPU measurement pass (run under gpurun): parity tests, bench line,
# ncu launch list of the bench command, per-launch DRAM traffic, and one
# full ncu capture of the dominant kernel.  Outputs land in gpurun_out/$TAG*.
TAG=${1:-r1}
CASE=${2:-"2048x512@70%/b128"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --cases-out gpurun_out/${TAG}_cases.json > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 600 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-compare --no-cpu > /dev/null 2>&1; echo ncu-launches $?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --nvtx --nvtx-include bench_timed/ -k regex:esc_spmm -c 90 --csv --log-file gpurun_out/${TAG}_dram.csv python bench.py --steps 1 --warmup 3 --no-compare --no-cpu > /dev/null 2>&1; echo ncu-dram $?; python tools/traffic_from_ncu.py gpurun_out/${TAG}_dram.csv gpurun_out/${TAG}_traffic.json suite
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include profile_reps/ -k regex:esc_spmm -c 1 -o gpurun_out/${TAG}_full python tools/profile_case.py --case "$CASE" --reps 3 > /dev/null 2>&1; echo ncu-full $?
