set -x
mkdir -p gpurun_out/final
timeout 300 python bench.py > gpurun_out/final/n1.json 2> gpurun_out/final/n1.err
timeout 300 python bench.py --no-fuse --no-engine-e2e > gpurun_out/final/n1_nofuse.json 2> gpurun_out/final/nofuse.err
for w in c1 c1lit c3 c4 c5 wc; do timeout 400 python bench.py --workload $w > gpurun_out/final/$w.json 2> gpurun_out/final/$w.err; done
timeout 300 python bench.py --impl reference > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 --no-engine-e2e --no-cpu-baseline > gpurun_out/final/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_segment_pass1 -s 5 -c 1 -o gpurun_out/final/ncu_fused python bench.py --steps 2 --warmup 3 --no-engine-e2e --no-cpu-baseline > gpurun_out/final/ncu_full.log 2>&1
ls -la gpurun_out/final
