# A/B: early mode with the next step triggered at the top (UCG_EARLY_TOP=1)
# against the default early mode; parity tests under the knob first
D=gpurun_out/r2t2; mkdir -p $D
UCG_EARLY_TOP=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fence.py -q -m gpu -x > $D/pytest_top.log 2>&1; echo "pytest top rc=$?"; tail -2 $D/pytest_top.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "consecutive or graph" > $D/pytest_default.log 2>&1; echo "pytest default rc=$?"; tail -2 $D/pytest_default.log
for rep in 1 2 3; do
  for e in "X=0" "UCG_EARLY_TOP=1"; do
    tag=$(echo $e | tr '=' '_')
    env $e timeout 600 python bench.py --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/c2_${tag}_$rep.json 2> $D/c2_${tag}_$rep.err
    env $e timeout 600 python bench.py --parts 8 --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/s8_${tag}_$rep.json 2> $D/s8_${tag}_$rep.err
    env $e timeout 600 python bench.py --workload c1 > $D/c1_${tag}_$rep.json 2> $D/c1_${tag}_$rep.err
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2t2/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], round(d.get("value")/1e9,2), round(d.get("ms_per_step")*1e3,2), (d.get("clocks") or {}).get("sm_mhz"), (d.get("parity") or {}).get("result_match"))
    except Exception as e: print(f, "ERR", e)
P
