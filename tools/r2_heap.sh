# seam-A chain under glibc allocator settings of the hosting process
T1="glibc.malloc.hugetlb=1"
T2="glibc.malloc.mmap_max=0:glibc.malloc.trim_threshold=68719476736"
T3="glibc.malloc.hugetlb=1:glibc.malloc.mmap_max=0:glibc.malloc.trim_threshold=68719476736"
for t in "" "$T1" "$T2" "$T3"; do echo "== GLIBC_TUNABLES=$t"; GLIBC_TUNABLES="$t" python tools/seam_a_breakdown.py --reps 3; done
for t in "" "$T3"; do echo "== ref_harness GLIBC_TUNABLES=$t"; GLIBC_TUNABLES="$t" ./oracle/_ref/ref_harness bench --parts 64 --part-len 16777216 --threads 16 --steps 2 --warmup 1; done
