# Sobel arithmetic forms at steady state: bench line (1 s soak + 20 steps) and
# 2000 back-to-back launches with clock/power, alternating; ncu of each form
D=gpurun_out/r2y; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "sobel" > $D/pytest_sobel.log 2>&1; echo "pytest rc=$?"
for rep in 1 2 3; do
  for a in half mix mix2 int; do
    UCG_SOBEL_ARITH=$a timeout 600 python bench.py --workload c4 > $D/c4_${a}_$rep.json 2> $D/c4_${a}_$rep.err
    UCG_SOBEL_ARITH=$a SOBEL_ITERS=2000 timeout 120 python tools/sobel_time.py | sed "s/^/{\"arith\": \"$a\", \"rep\": $rep, \"line\": /; s/$/}/" >> $D/steady.jsonl
  done
done
for a in half mix mix2; do
  UCG_SOBEL_ARITH=$a timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sobel_tma -c 1 -o $D/ncu_$a python tools/sobel_time.py > $D/ncu_$a.log 2>&1; echo "ncu $a rc=$?"
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2y/c4_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], round(d["ms_per_step"]*1e3,2), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])
for l in open("gpurun_out/r2y/steady.jsonl"):
    d=json.loads(l); print(d["arith"], d["rep"], round(d["line"]["us"],2), d["line"]["sm_mhz_median"], d["line"]["watts_median"], d["line"]["md5"][:8])
P
