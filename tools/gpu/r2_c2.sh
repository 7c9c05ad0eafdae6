set -x
python -m paper_1903_12359_b200.build
timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_cfg2.py -p no:cacheprovider > gpurun_out/r2_tests_c2.log 2>&1
tail -15 gpurun_out/r2_tests_c2.log
