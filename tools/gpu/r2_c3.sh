set -x
python -m paper_1903_12359_b200.build
timeout 900 python -m pytest tests/test_gpu_cfg2.py -m gpu -q -s -p no:cacheprovider > gpurun_out/r2_cfg2_tests.log 2>&1
tail -15 gpurun_out/r2_cfg2_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
tail -3 gpurun_out/r2_bench_c3.err
cat gpurun_out/r2_bench_c3.json
