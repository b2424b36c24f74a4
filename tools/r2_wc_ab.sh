# word flags: self-resetting claim pair (no memset launch) and 4 KB blocks (UCG_WC_WU=8) A/B
D=gpurun_out/r2wc; mkdir -p $D
for w in 4 8; do UCG_WC_WU=$w timeout 600 python -m pytest tests/test_wordcount.py -q -m gpu > $D/pytest_wu$w.log 2>&1; echo "pytest wu$w rc=$?"; tail -1 $D/pytest_wu$w.log; done
for rep in 1 2 3; do for w in 4 8; do
  UCG_WC_WU=$w timeout 600 python bench.py --workload wc > $D/wc_wu${w}_$rep.json 2> $D/wc_wu${w}_$rep.err
done; done
UCG_WC_WU=8 timeout 600 ncu --set full --clock-control none -k regex:k_word_flags -c 1 -o $D/ncu_wc_wu8 python bench.py --workload wc --steps 2 --warmup 3 > $D/ncu.log 2>&1; echo "ncu rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2wc/wc_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], round(d["value"]/1e12,3), round(d["ms_per_step"]*1e3,1), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])
P
