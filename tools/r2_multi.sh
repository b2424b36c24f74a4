nvidia-smi -L
timeout 900 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -s > gpurun_out/r2e_pytest_multigpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_pytest_multigpu.log
tail -3 gpurun_out/r2e_pytest_multigpu.log
N=$(nvidia-smi -L | wc -l)
timeout 900 python bench.py --gpus $N > gpurun_out/r2e_bench_n$N.json 2> gpurun_out/r2e_bench_n$N.err; echo "bench rc=$?"
timeout 900 python bench.py --gpus 2 > gpurun_out/r2e_bench_n2.json 2> gpurun_out/r2e_bench_n2.err; echo "bench2 rc=$?"
timeout 900 python bench.py --gpus $N --parts $((8*N)) > gpurun_out/r2e_bench_shard8_n$N.json 2> gpurun_out/r2e_bench_shard8_n$N.err
python - <<P
import json,glob
for f in sorted(glob.glob("gpurun_out/r2e_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["n_gpus"], d["value"]/1e9, d["ms_per_step"], d["roofline"]["frac"], (d.get("cpu_baseline") or {}).get("value"), (d.get("parity") or {}).get("result_match"), d["e2e"]["value"]/1e9)
    except Exception as e: print(f, "ERR", e)
P
