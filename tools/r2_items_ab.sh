for rep in 1 2; do
for L in 12 11 10 13; do
  UCG_ITEM_LOG2=$L timeout 600 python bench.py --parts 8 --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 50 > gpurun_out/r2n_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2n_ab.json').read().strip().splitlines()[-1]);print('item_log2=$L parts=8 rep=$rep', round(d['ms_per_step']*1e3,2), 'us/step')"
  UCG_ITEM_LOG2=$L timeout 600 python bench.py --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 20 > gpurun_out/r2n_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2n_ab.json').read().strip().splitlines()[-1]);print('item_log2=$L parts=64 rep=$rep', round(d['ms_per_step']*1e3,2), 'us/step')"
done
done
