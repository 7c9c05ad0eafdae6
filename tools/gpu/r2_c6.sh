python -m paper_1903_12359_b200.build
for i in 1 2; do
  PGCP_HARM_ORDER=0 python bench.py --steps 5 --warmup 3 --no-cfg5 --no-cpu-baseline --no-e2e > gpurun_out/r2_ab_horder0_$i.json 2>/dev/null
  python bench.py --steps 5 --warmup 3 --no-cfg5 --no-cpu-baseline --no-e2e > gpurun_out/r2_ab_horder1_$i.json 2>/dev/null
done
python - <<'PY'
import json
for tag in ("horder0", "horder1"):
    for i in (1, 2):
        d = json.load(open(f"gpurun_out/r2_ab_{tag}_{i}.json"))
        print(tag, i, round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["stages_ms_per_step"].items() if k in ("harmonic", "flatten", "weld")})
PY
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -p no:cacheprovider > gpurun_out/r2_fullsize.log 2>&1
grep -E "^\[cfg|passed|failed|Error|assert" gpurun_out/r2_fullsize.log | head -20
