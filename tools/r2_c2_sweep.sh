# C2 pass-1 variant and item-size sweep under the early-stream mode (2^30 and the 8-GPU shard size)
D=gpurun_out/r2cs; mkdir -p $D
for rep in 1 2; do
  for v in 0 1 2 5; do
    UCG_PASS1_VARIANT=$v timeout 600 python bench.py --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/c2_v${v}_$rep.json 2> /dev/null
    UCG_PASS1_VARIANT=$v timeout 600 python bench.py --parts 8 --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/s8_v${v}_$rep.json 2> /dev/null
  done
  for l in 11 13; do
    UCG_ITEM_LOG2=$l timeout 600 python bench.py --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/c2_L${l}_$rep.json 2> /dev/null
    UCG_ITEM_LOG2=$l timeout 600 python bench.py --parts 8 --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/s8_L${l}_$rep.json 2> /dev/null
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2cs/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], round(d["value"]/1e9,2), round(d["ms_per_step"]*1e3,2), (d.get("parity") or {}).get("result_match"))
    except Exception as e: print(f, "ERR", e)
P
