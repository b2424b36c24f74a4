# Workload lines after the soak change; Sobel int vs fp16 arithmetic over 2000
# back-to-back launches with SM clock / power sampled (is the fp16 form power-capped?)
D=gpurun_out/r2v; mkdir -p $D
for w in c4 wc c3 c1; do timeout 600 python bench.py --workload $w > $D/$w.json 2> $D/$w.err; echo "$w rc=$?"; done
for rep in 1 2; do
  for a in int half; do
    UCG_SOBEL_ARITH=$a SOBEL_ITERS=2000 timeout 120 python tools/sobel_time.py | sed "s/^/{\"arith\": \"$a\", \"rep\": $rep, \"line\": /; s/$/}/" >> $D/power.jsonl
  done
done
timeout 900 python bench.py --workload c5 > $D/c5.json 2> $D/c5.err; echo "c5 rc=$?"
cat $D/power.jsonl
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2v/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("unit"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), d.get("clocks"))
    except Exception as e: print(f, "ERR", e)
P
