# final-tree multi-GPU pass after the e2e transfer overlap changes (same steps as r2_multi_final.sh)
# pipeline at N ranks, the C++ drop-in over N GPUs), every workload at
# --gpus N, the 8-GPU shard size at N ranks, and C2 at 2 and N
N=$(nvidia-smi -L | wc -l)
D=gpurun_out/r2m3; mkdir -p $D
timeout 1500 python -m pytest tests -q -m gpu > $D/pytest_gpu_n$N.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest_gpu_n$N.log
for w in c2 c1 c3 c4 c5 wc; do timeout 900 python bench.py --gpus $N --workload $w --no-tuned-heap > $D/${w}_n$N.json 2> $D/${w}_n$N.err; echo "$w rc=$?"; done
timeout 900 python bench.py --gpus $N --parts $((8*N)) --no-engine-e2e --no-tuned-heap > $D/shard8_n$N.json 2> $D/shard8_n$N.err; echo "shard8 rc=$?"
timeout 900 python bench.py --gpus 2 --no-tuned-heap > $D/c2_n2.json 2> $D/c2_n2.err; echo "c2 n2 rc=$?"
timeout 900 python bench.py --gpus 2 --parts 16 --no-engine-e2e --no-tuned-heap > $D/shard8_n2.json 2> $D/shard8_n2.err; echo "shard8 n2 rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2m3/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], d["n_gpus"], d["value"], d["unit"], d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"), (d.get("parity") or {}).get("result_match"))
    except Exception as e: print(f, "ERR", e)
P
