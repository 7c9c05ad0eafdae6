python -m paper_1903_12359_b200.build
python tools/l2_probe_sweep.py > gpurun_out/r2_l2_probe2.log 2>&1; cat gpurun_out/r2_l2_probe2.log
python tools/l2_probe_sweep.py > gpurun_out/r2_l2_probe3.log 2>&1; cat gpurun_out/r2_l2_probe3.log
