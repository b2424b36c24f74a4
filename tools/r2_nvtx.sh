# NVTX ranges seen by ncu: kernels launched inside DeviceEngine's map_cl_partition:psum range of the C++ drop-in test
D=gpurun_out/r2nv; mkdir -p $D
timeout 600 ncu --nvtx --nvtx-include "ucores.map_cl_partition:psum/" --metrics gpu__time_duration.sum -c 3 build/test_dropin > $D/ncu_nvtx.txt 2>&1; echo "ncu rc=$?"
grep -E 'NVTX|ucores|k_segment|Duration|==PROF==|RESULT' $D/ncu_nvtx.txt | head -30
