# Sobel: row-streaming kernel (terms once per input row) vs TMA tiles, both in
# the mixed arithmetic, at steady state; parity of the row kernel's forms
D=gpurun_out/r2r; mkdir -p $D
for a in mix half mix2 int; do UCG_SOBEL_VARIANT=0 UCG_SOBEL_ARITH=$a timeout 300 python tests/sobel_variant_worker.py > $D/parity_rows_$a.json 2>&1; echo "parity rows $a rc=$?"; cat $D/parity_rows_$a.json | tail -1; done
for rep in 1 2 3; do
  for v in 1 0; do
    UCG_SOBEL_VARIANT=$v timeout 600 python bench.py --workload c4 > $D/c4_v${v}_$rep.json 2> $D/c4_v${v}_$rep.err
    UCG_SOBEL_VARIANT=$v SOBEL_ITERS=2000 timeout 120 python tools/sobel_time.py | sed "s/^/{\"v\": $v, \"rep\": $rep, \"line\": /; s/$/}/" >> $D/steady.jsonl
  done
done
UCG_SOBEL_VARIANT=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sobel_rows -c 1 -o $D/ncu_rows_mix python tools/sobel_time.py > $D/ncu_rows.log 2>&1; echo "ncu rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2r/c4_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], round(d["ms_per_step"]*1e3,2), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])
for l in open("gpurun_out/r2r/steady.jsonl"):
    d=json.loads(l); print(d["v"], d["rep"], round(d["line"]["us"],2), d["line"]["sm_mhz_median"], d["line"]["md5"][:8])
P
