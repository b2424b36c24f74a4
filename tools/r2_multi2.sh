# round-2 multi-GPU pass: the C++ drop-in (seam A / seam B / DeviceEngine
# over every visible GPU), the sharded pipeline test, and every workload's
# bench line at N GPUs through the self-launching bench.py
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out/r2j
timeout 900 python -m pytest tests/test_cpp_dropin.py tests/test_multigpu.py -q -p no:cacheprovider -s > gpurun_out/r2j/pytest_n$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2j/pytest_n$N.log
for w in c2 c1 c3 c4 c5 wc; do timeout 900 python bench.py --gpus $N --workload $w --no-tuned-heap > gpurun_out/r2j/${w}_n$N.json 2> gpurun_out/r2j/${w}_n$N.err; echo "$w rc=$?"; done
timeout 900 python bench.py --gpus $N --parts $((8*N)) --no-engine-e2e > gpurun_out/r2j/shard8_n$N.json 2> gpurun_out/r2j/shard8_n$N.err; echo "shard8 rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2j/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["n_gpus"], d["value"], d["unit"], d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e: print(f, "ERR", e)
P
