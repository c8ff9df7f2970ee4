#!/bin/bash
# Round-end GPU pass (run under gpurun): smoke, full GPU tests, default bench line,
# C4/C5/ResNet-50 lines, ncu launch list + DRAM bytes of the timed region only.
TAG=${1:-r1f}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --cases-out gpurun_out/${TAG}_cases.json > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 400 gpurun_out/${TAG}_bench.json; tail -2 gpurun_out/${TAG}_bench.err
for w in c4 c5 resnet50; do
  timeout 900 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
  tail -c 200 gpurun_out/${TAG}_bench_$w.json; echo
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include bench_timed/ --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-compare --no-cpu > /dev/null 2>&1; echo ncu-launches $?
