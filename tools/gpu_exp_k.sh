# kernel A/B (gpurun): pytest gpu, then bench each env variant on $CONFIGS (default "3 5")
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_k.log
for v in "$@"; do
  for c in ${CONFIGS:-3 5}; do
    env $v python bench.py --no-cpu-baseline --e2e-steps 1 --config $c > gpurun_out/k${c}_$(echo $v | tr '= ' '__').json 2>> gpurun_out/k.log
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/k[0-9]_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "value", round(d["value"]), "kernel_ms", round(d["roofline"]["kernel_ms"], 4), "frac", round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(f, "ERR", e)
PY
