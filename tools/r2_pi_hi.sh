# pi: SplitMix64 high-word shifts on the FMA pipe (UCG_PI_HI bit mask), parity then A/B
D=gpurun_out/r2pi; mkdir -p $D
for m in 0 1 3 7; do UCG_PI_HI=$m timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -k "pi" > $D/pytest_$m.log 2>&1; echo "pytest $m rc=$?"; tail -1 $D/pytest_$m.log; done
for rep in 1 2; do for m in 0 1 3 7; do
  UCG_PI_HI=$m timeout 600 python bench.py --workload c3 > $D/c3_${m}_$rep.json 2> $D/c3_${m}_$rep.err
done; done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2pi/c3_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], round(d["value"]/1e9,2), round(d["ms_per_step"],3), d["clocks"]["sm_mhz"], d["config"].get("hits_total"))
P
