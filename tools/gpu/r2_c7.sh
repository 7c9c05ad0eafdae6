python -m paper_1903_12359_b200.build
( time timeout 1200 python -m pytest tests/test_gpu_fullsize.py -k cfg5 -q -s -p no:cacheprovider ) > gpurun_out/r2_fullsize_cfg5.log 2>&1
grep -E "^\[cfg|passed|failed|Error|assert|real" gpurun_out/r2_fullsize_cfg5.log | head
PGCP_BENCH_DIST=1 timeout 600 python bench.py --steps 3 --warmup 2 > gpurun_out/r2_bench_dist1.json 2> gpurun_out/r2_bench_dist1.err
tail -2 gpurun_out/r2_bench_dist1.err; cut -c 1-600 gpurun_out/r2_bench_dist1.json; grep -o '"exchanged_bytes_per_step": [0-9.]*' gpurun_out/r2_bench_dist1.json
PGCP_PCG_TIMING=1 timeout 300 python tools/hprep_time.py > gpurun_out/r2_pcg_timing.log 2>&1
grep -E "build_system|prepare|flatten call" gpurun_out/r2_pcg_timing.log | head -12
