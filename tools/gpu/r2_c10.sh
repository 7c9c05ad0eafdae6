python -m paper_1903_12359_b200.build
for nt in 512 1024 512 1024; do
  echo "NT=$nt"; PGCP_PCG2_NT=$nt timeout 300 python tools/hprep_time.py 2>&1 | tail -2
done
PGCP_PCG2_NT=1024 timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x -k "pipeline_matches or determinism" -p no:cacheprovider 2>&1 | tail -2
PGCP_PCG2_NT=1024 timeout 300 python tools/cfg5_flatten.py 2>&1 | tail -1
