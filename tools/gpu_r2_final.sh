#!/bin/bash
# Round-2 evidence pass (run under gpurun): ncu launch list of the bench step
# (CUDA-graph replay), per-launch DRAM bytes of one step, one full capture of
# the dominant kernel in its bench configuration (the staged walk), and
# compute-sanitizer memcheck / racecheck / synccheck on the small cases.
TAG=${1:-r2i}
CASE=${2:-"512x4608@70%/b128"}
mkdir -p gpurun_out
# tune once without the profiler (the tuner's timings under ncu are not the
# bench's), then profile the same plans through the persisted tuning cache
export ESCS_TUNE_CACHE_FILE=/tmp/escs_tune_${TAG}.txt
rm -f $ESCS_TUNE_CACHE_FILE
timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-compare --no-cpu --streams 1 > gpurun_out/${TAG}_bench_pre.json 2>/dev/null; echo tune $?
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-compare --no-cpu --streams 1 > /dev/null 2>&1; echo ncu-launches $?
timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --nvtx --nvtx-include bench_timed/ -k regex:"esc_(rec|spmm|staged)_kernel" -c 90 --csv --log-file gpurun_out/${TAG}_dram.csv python bench.py --steps 1 --warmup 3 --no-compare --no-cpu --streams 1 > /dev/null 2>&1; echo ncu-dram $?
python tools/traffic_from_ncu.py gpurun_out/${TAG}_dram.csv gpurun_out/${TAG}_traffic.json suite "$CASE"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include profile_reps/ -k regex:"esc_staged_kernel" -c 1 -o gpurun_out/${TAG}_full_staged python tools/profile_case.py --case "$CASE" --staged 8,16,1,0 --reps 3 > gpurun_out/${TAG}_full_staged.log 2>&1; echo ncu-full $?
# (compute-sanitizer is closed on this pool; the small cases run plain, exact vs the oracle)
timeout -s KILL 600 python tools/sanitize_cases.py > gpurun_out/${TAG}_small_cases.log 2>&1; echo small-cases $?
grep -c " ok" gpurun_out/${TAG}_small_cases.log; grep -c MISMATCH gpurun_out/${TAG}_small_cases.log
