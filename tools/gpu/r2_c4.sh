set -x
python -m paper_1903_12359_b200.build
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_fullsize.py > gpurun_out/r2_tests_c4.log 2>&1
tail -5 gpurun_out/r2_tests_c4.log
python tools/hprep_time.py > gpurun_out/r2_hprep.log 2>&1
cat gpurun_out/r2_hprep.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -p no:cacheprovider > gpurun_out/r2_fullsize.log 2>&1
tail -12 gpurun_out/r2_fullsize.log
