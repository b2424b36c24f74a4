# Early-stream mode A/B (consecutive steps overlap stream and previous tail)
# + Sobel arithmetic A/B in the bench's steady state. Same box, alternating.
D=gpurun_out/r2w; mkdir -p $D
timeout 1500 python -m pytest tests -q -m gpu -x > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"
for rep in 1 2 3; do
  for e in "X=0" "UCG_NO_EARLY=1"; do
    tag=$(echo $e | tr '=' '_')
    env $e timeout 600 python bench.py --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/c2_${tag}_$rep.json 2> $D/c2_${tag}_$rep.err
    env $e timeout 600 python bench.py --parts 8 --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/s8_${tag}_$rep.json 2> $D/s8_${tag}_$rep.err
    env $e timeout 600 python bench.py --workload c1 > $D/c1_${tag}_$rep.json 2> $D/c1_${tag}_$rep.err
  done
  for a in int half; do
    UCG_SOBEL_ARITH=$a timeout 600 python bench.py --workload c4 > $D/c4_${a}_$rep.json 2> $D/c4_${a}_$rep.err
    UCG_SOBEL_ARITH=$a SOBEL_ITERS=2000 timeout 120 python tools/sobel_time.py | sed "s/^/{\"arith\": \"$a\", \"rep\": $rep, \"line\": /; s/$/}/" >> $D/sobel_power.jsonl
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2w/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], round(d.get("value")/1e9,2), d.get("ms_per_step"), round((d.get("roofline") or {}).get("frac") or 0,4), (d.get("clocks") or {}).get("sm_mhz"), (d.get("parity") or {}).get("result_match"))
    except Exception as e: print(f, "ERR", e)
P
cat $D/sobel_power.jsonl
