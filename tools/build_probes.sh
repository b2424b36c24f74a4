#!/bin/bash
# Host-side probes (not the product): tools/host_copy_probe.cpp, tools/pipe_probe.cpp
set -e
cd "$(dirname "$0")/.."
mkdir -p build
g++ -O2 -std=c++20 -pthread tools/host_copy_probe.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -o build/host_copy_probe
g++ -O2 -std=c++20 -pthread tools/pipe_probe.cpp -I/root/reference/proj/include -Iinclude -Ipaper_1505_01120_b200/host \
  -I/usr/local/cuda/include -Lpaper_1505_01120_b200/_lib -lucores_cuda -Wl,-rpath,'$ORIGIN/../paper_1505_01120_b200/_lib' \
  -L/usr/local/cuda/lib64 -lcudart -o build/pipe_probe
JSON_INC=$(python3 -c "import os,sysconfig;print(os.path.join(sysconfig.get_paths()['purelib'],'include','cudnn_frontend','thirdparty','nlohmann'))")
g++ -O2 -std=c++20 -pthread -ffp-contract=off tools/literal_probe.cpp -I/root/reference/proj/include -I$JSON_INC -Iinclude \
  -Ipaper_1505_01120_b200/host -I/usr/local/cuda/include -Lpaper_1505_01120_b200/_lib -lucores_cuda \
  -Wl,-rpath,'$ORIGIN/../paper_1505_01120_b200/_lib' -L/usr/local/cuda/lib64 -lcudart -o build/literal_probe
