# last check of the final tree on one GPU: whole GPU suite, smoke, default bench line, word flags and C5 lines
D=gpurun_out/r2z5; mkdir -p $D
timeout 1800 python -m pytest tests -q -m gpu > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $D/smoke.log
timeout 900 python bench.py > $D/n1.json 2> $D/n1.err; echo "bench rc=$?"
for w in wc c5 c4 c1; do timeout 900 python bench.py --workload $w > $D/$w.json 2> $D/$w.err; echo "$w rc=$?"; done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2z5/*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], d["value"], d["unit"], d["ms_per_step"], (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("sm_mhz"), d.get("step_overlap","")[:30])
P
