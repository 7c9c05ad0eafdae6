# round-2 late diagnostics: per-phase / per-level split of the direct solver,
# weld timing, the NCCL bench path at world size 1, and --set full captures
# of the two top kernels of the step (k_factor_warp, k_phase1w).
mkdir -p gpurun_out
PGCP_DIRECT_TIMING=2 timeout 300 python tools/direct_prof.py > gpurun_out/direct_prof.log 2>&1; echo "direct_prof $?"
PGCP_WELD_TIMING=1 timeout 300 python tools/weld_timing.py > gpurun_out/weld_timing.log 2>&1; echo "weld_timing $?"
PGCP_BENCH_DIST=1 timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; echo "dist bench $?"
HARMONIC=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_factor_warp -c 5 -o gpurun_out/r2_factor_warp -f python tools/direct_once.py > gpurun_out/ncu_fw.log 2>&1; echo "ncu fw $?"
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_phase1w -c 6 -o gpurun_out/r2_phase1w -f python tools/prof_weld.py > gpurun_out/ncu_w.log 2>&1; echo "ncu weld $?"
