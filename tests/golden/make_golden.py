"""Regenerate tests/golden/ref_golden.json from the UNMODIFIED reference.

Builds oracle/_ref/ref_harness from the reference headers under
/root/reference/proj/include (oracle/Makefile) and records its `golden`
output. Only runnable where the reference tree exists (this container); the
committed JSON is what travels.
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
    out = subprocess.run([str(exe), "golden"], check=True, capture_output=True, text=True).stdout
    data = json.loads(out)
    (ROOT / "tests" / "golden" / "ref_golden.json").write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print("wrote", ROOT / "tests" / "golden" / "ref_golden.json")
    return 0


if __name__ == "__main__":
    sys.exit(main())
