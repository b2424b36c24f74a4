# Same-box A/B of two builds of libucores_cuda.so on one workload:
#   bash tools/lib_ab.sh build/variant.so sobel
L=paper_1505_01120_b200/_lib/libucores_cuda.so
cp $L /tmp/base.so
for rep in 1 2 3; do
  cp /tmp/base.so $L; echo "base    $(timeout 200 python tools/ab_time.py $2 X=1 2>&1 | tail -1)"
  cp $1 $L; echo "variant $(timeout 200 python tools/ab_time.py $2 X=1 2>&1 | tail -1)"
done
cp /tmp/base.so $L
