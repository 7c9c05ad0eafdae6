# A/B of the harmonic-preparation placement after the pinned-staging fix, the
# NCCL bench path at world size 1, and the FP64 latency microbenchmarks.
mkdir -p gpurun_out
B="python bench.py --no-pcg --no-cfg5 --no-cpu-baseline --steps 10 --warmup 3"
for i in 1 2; do
  timeout 200 $B 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('flatten-placed', d['ms_per_step'], d['e2e']['ms_per_step'], d['stages_ms_per_step'])"
  PGCP_HPREP_AT=weld timeout 200 $B 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('weld-placed   ', d['ms_per_step'], d['e2e']['ms_per_step'], d['stages_ms_per_step'])"
done
PGCP_BENCH_DIST=1 timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; echo "dist bench $?"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gpu/fp64_latency.cu -o /tmp/fp64_lat && /tmp/fp64_lat > gpurun_out/fp64_latency.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gpu/open_chain.cu -o /tmp/oc && /tmp/oc > gpurun_out/open_chain.log 2>&1
