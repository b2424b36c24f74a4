# e2e of C4 and word flags with uploads overlapping downloads (pieces)
D=gpurun_out/r2dx; mkdir -p $D
for w in c5 c4 wc; do timeout 900 python bench.py --workload $w > $D/$w.json 2> $D/$w.err; echo "$w rc=$?"; done
python - <<'P'
import json
for w in ["c5","c4","wc"]:
    d=json.loads(open(f"gpurun_out/r2dx/{w}.json").read().strip().splitlines()[-1])
    print(w, d["value"], d["e2e"])
P
