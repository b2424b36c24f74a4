# two ranks on one GPU through the fused exchange (time-sliced contexts)
D=gpurun_out/r2sg; mkdir -p $D
nvidia-smi --query-gpu=compute_mode --format=csv > $D/compute_mode.txt
( time timeout 400 python -m pytest tests/test_multigpu.py -q -m gpu -s -k ranks_one_gpu ) > $D/pytest_shared.log 2>&1; echo "shared rc=$?"; tail -5 $D/pytest_shared.log
