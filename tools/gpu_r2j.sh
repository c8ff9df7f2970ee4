#!/bin/bash
# Round-2 final pass (run under gpurun): smoke, every GPU test file, the bench
# lines (suite with the per-case table, --ufi 4, C4, C5).
TAG=${1:-r2j}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for f in tests/test_gpu_staged.py tests/test_gpu_hybrid.py tests/test_gpu_records.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_abi.py tests/test_c_client.py tests/test_dist.py; do
  timeout -s KILL 900 python -m pytest $f -m gpu -q -x 2>&1 | tail -1
done
timeout -s KILL 1200 python bench.py --cases-out gpurun_out/${TAG}_cases_suite.json > gpurun_out/${TAG}_bench_suite.json 2> gpurun_out/${TAG}_bench_suite.err; echo bench $?
timeout -s KILL 900 python bench.py --workload c4 --cases-out gpurun_out/${TAG}_cases_c4.json > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err; echo c4 $?
timeout -s KILL 1500 python bench.py --workload c5 --no-compare > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err; echo c5 $?
timeout -s KILL 900 python bench.py --ufi 4 --no-compare --no-cpu > gpurun_out/${TAG}_bench_suite_ufi4.json 2> /dev/null; echo ufi4 $?
python tools/bench_summary.py gpurun_out/${TAG}_bench_*.json
