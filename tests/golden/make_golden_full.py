"""Regenerate tests/golden/ref_golden_full.json: the UNMODIFIED reference's own
results at the BASELINE.json sizes (oracle/_ref/ref_harness golden-full —
reference Engine + WorkerRuntime + HostParallelExecutor over the workload
kernels written in the reference API):

  c2_full  2^30 fp32 in 64 partitions (partition p from seed 1000+p, planted
           maximum 1.5 in partition 32 at index 2^24/3): per-partition FNV-1a
           of y = map_cl(axpb), all 64 psum/pmax partials, reduce_cl sum2/max2
  c3_full  pi, 2^34 samples in 64 tasks of 2^28 (seed 42+t): all 64 hit counts
  c4_full  Sobel 16384^2 u8 (seed 7) in 64 bands of 256 rows: per-band FNV-1a

Takes ~2.5 min on 8 host threads and ~16 GB of RAM. Only runnable where the
reference tree exists (this container); the committed JSON is what travels.
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]


def main() -> int:
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)
    exe = ROOT / "oracle" / "_ref" / "ref_harness"
    if not exe.exists():
        print("reference tree absent; cannot regenerate goldens", file=sys.stderr)
        return 1
    data = {}
    for which in ("c2", "c3", "c4"):
        out = subprocess.run([str(exe), "golden-full", "--which", which], check=True, capture_output=True,
                             text=True).stdout
        data.update(json.loads(out))
    dst = ROOT / "tests" / "golden" / "ref_golden_full.json"
    dst.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print("wrote", dst)
    return 0


if __name__ == "__main__":
    sys.exit(main())
