# full bench line on HEAD, launch list, and a --set full capture of the
# size-grouped k_factor_warp
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_step5.json 2> gpurun_out/bench_step5.err; echo "bench $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-pcg --no-cfg5 --no-cpu-baseline > gpurun_out/ncu_bench5.log 2>&1; echo "ncu list $?"
HARMONIC=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_factor_warp -c 6 -o gpurun_out/r2_factor_warp_grouped -f python tools/direct_once.py > gpurun_out/ncu_fw5.log 2>&1; echo "ncu fw $?"
