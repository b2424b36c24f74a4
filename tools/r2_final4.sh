# last check of the final tree on one GPU: the whole GPU suite, smoke, the default bench line
D=gpurun_out/r2z4; mkdir -p $D
timeout 1800 python -m pytest tests -q -m gpu > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $D/smoke.log
timeout 900 python bench.py > $D/n1.json 2> $D/n1.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$D/n1.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'], d['parity']['result_match'], d['gpu_launches'])"
