# end-of-round validation on HEAD: smoke, the whole GPU suite, the default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
(timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_final.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputests_final.log); tail -3 gpurun_out/gputests_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference arm $?"
PGCP_BENCH_DIST=1 timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_dist_final.json 2> gpurun_out/bench_dist_final.err; echo "dist bench $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-pcg --no-cfg5 --no-cpu-baseline > gpurun_out/ncu_bench_final.log 2>&1; echo "ncu list $?"
