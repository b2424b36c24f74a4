D=gpurun_out/r2c1; mkdir -p $D
for rep in 1 2; do for c in 1 4; do UCG_C1_E2E_CHUNKS=$c timeout 600 python bench.py --workload c1 > $D/c1_ch${c}_$rep.json 2> $D/c1_ch${c}_$rep.err; done; done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2c1/*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d["value"]/1e9,1), round(d["e2e"]["value"]/1e9,2))
P
