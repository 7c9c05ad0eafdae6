python -m paper_1903_12359_b200.build
python tools/l2_probe_sweep.py > gpurun_out/r2_l2_probe.log 2>&1; cat gpurun_out/r2_l2_probe.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c8.json 2> gpurun_out/r2_bench_c8.err
tail -2 gpurun_out/r2_bench_c8.err; cut -c 1-300 gpurun_out/r2_bench_c8.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; cut -c 1-300 gpurun_out/r2_bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --no-cfg5 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_launch.log 2>&1
tail -2 gpurun_out/r2_ncu_launch.log
python tools/summarize_launches.py gpurun_out/r2_launches.csv 1 > gpurun_out/r2_launches_summary.json; head -c 1500 gpurun_out/r2_launches_summary.json
