for rep in 1 2; do
for v in "UCG_TAGGED_TAIL=1" "UCG_TAGGED_TAIL=1 UCG_TAGGED_LAST=1" "UCG_TAGGED_TAIL=0"; do
  env $v timeout 600 python bench.py --parts 8 --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 50 > gpurun_out/r2k_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2k_ab.json').read().strip().splitlines()[-1]);print('$v rep=$rep', round(d['ms_per_step']*1e3,2), 'us/step kernel', round(d['roofline']['kernel_ms']*1e3,2), d['result'])"
done
done
UCG_TAGGED_TAIL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_segment_pass1 -s 8 -c 1 -o gpurun_out/r2k_ncu_tagged python bench.py --parts 8 --steps 3 --warmup 3 --no-engine-e2e --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
UCG_TAGGED_TAIL=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_segment_pass1 -s 8 -c 1 -o gpurun_out/r2k_ncu_ticketed python bench.py --parts 8 --steps 3 --warmup 3 --no-engine-e2e --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls gpurun_out/r2k_ncu*
