# every workload at N=2 and N=4 (one 4-GPU box): lines into gpurun_out/sweep/
mkdir -p gpurun_out/sweep
port=29600
for N in 2 4; do
  for w in c2 c1 c3 c4 c5 wc; do
    port=$((port+1))
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N --workload $w > gpurun_out/sweep/${w}_n$N.json 2> gpurun_out/sweep/${w}_n$N.err
    echo "$w N=$N rc=$?"
  done
done
