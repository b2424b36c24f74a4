# Early-stream mode on 2+ GPUs: multi-GPU parity tests, then C2 lines with and
# without it (2^30 total, and the 8-GPU shard size per rank), alternating
D=gpurun_out/r2x4; mkdir -p $D
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py tests/test_gpu_parity.py -q -m gpu -x -k "multigpu or sharded or consecutive or graph" > $D/pytest_multi.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest_multi.log
for rep in 1 2 3; do
  for e in "X=0" "UCG_EARLY_LATE_TRIGGER=1"; do
    tag=$(echo $e | tr '=' '_')
    env $e timeout 600 python bench.py --gpus $N --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/c2_n${N}_${tag}_$rep.json 2> $D/c2_n${N}_${tag}_$rep.err
    env $e timeout 600 python bench.py --gpus $N --parts $((8 * N)) --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/s8_n${N}_${tag}_$rep.json 2> $D/s8_n${N}_${tag}_$rep.err
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2x4/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], d.get("n_gpus"), round(d.get("value")/1e9,2), round(d.get("ms_per_step")*1e3,2), (d.get("parity") or {}).get("result_match"))
    except Exception as e: print(f, "ERR", e)
P
