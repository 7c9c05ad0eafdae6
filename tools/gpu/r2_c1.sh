set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_1903_12359_b200.build
python tools/cfg5_flatten.py > gpurun_out/r2_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pcg2 -c 1 -o gpurun_out/r2_cfg5_pcg2 -f python tools/cfg5_flatten.py > gpurun_out/r2_cfg5_ncu.log 2>&1
tail -3 gpurun_out/r2_cfg5_ncu.log
