timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest_gpu.log
tail -3 gpurun_out/r2c_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2c_bench_n1.json 2> gpurun_out/r2c_bench_n1.err
timeout 600 python bench.py --workload c1lit > gpurun_out/r2c_bench_c1lit.json 2> gpurun_out/r2c_bench_c1lit.err
python - <<'P'
import json
for f in ["gpurun_out/r2c_bench_n1.json","gpurun_out/r2c_bench_c1lit.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), json.dumps(d.get("e2e_reference_api"))[:1500], d.get("cpu_baseline"))
    except Exception as e: print(f, e)
P
