# end-of-round validation on HEAD: smoke, the whole GPU suite, the default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
(timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_final.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputests_final.log); tail -3 gpurun_out/gputests_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference arm $?"
