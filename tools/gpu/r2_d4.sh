# --set full captures after the session's changes: the size-grouped
# k_factor_warp on the leaf-side levels (skip the small top launches) and the
# streamed replay beside phase 1
mkdir -p gpurun_out
HARMONIC=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_factor_warp -s 6 -c 8 -o gpurun_out/r2_factor_warp_grouped -f python tools/direct_once.py > gpurun_out/ncu_fw6.log 2>&1; echo "ncu fw $?"
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_replay_stream -c 6 -o gpurun_out/r2_replay_stream -f python tools/prof_weld.py > gpurun_out/ncu_rs.log 2>&1; echo "ncu replay $?"
