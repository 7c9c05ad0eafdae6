python -m paper_1903_12359_b200.build
timeout 600 python -m pytest tests/test_gpu_fullsize.py -k cfg3 -x -q -s --tb=long -p no:cacheprovider > gpurun_out/r2_fullsize_cfg3.log 2>&1
tail -60 gpurun_out/r2_fullsize_cfg3.log
