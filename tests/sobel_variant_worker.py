"""Subprocess worker for tests/test_gpu_parity.py::test_sobel_kernel_variants:
the Sobel kernel variant is fixed per process (UCG_SOBEL_VARIANT /
UCG_SOBEL_ARITH are read once), so each variant runs in its own process and
compares every case against the C oracle (orc_sobel_band_u8). Prints one JSON
line {"variant", "arith", "cases", "bad"}."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402
from paper_1505_01120_b200 import capi, ops  # noqa: E402


def images():
    # random images at widths that take the vectorised paths (multiples of 16)
    for (H, W, rows, seed) in [(50, 48, 16, 7), (64, 256, 32, 3), (37, 1024, 5, 9), (300, 528, 64, 1),
                               (130, 4096, 64, 11), (67, 272, 67, 4)]:
        yield f"rand{H}x{W}/{rows}", O.sobel_image(H, W, seed), rows
    # extremes: |Gx|+|Gy| up to 2040 (checkerboards, stripes, a single hot
    # pixel, flat 255), where a lost bit in the packed arithmetic would show
    H, W = 96, 512
    y, x = np.mgrid[0:H, 0:W]
    pats = {
        "checker": ((x + y) & 1) * 255,
        "checker2": (((x >> 1) + (y >> 1)) & 1) * 255,
        "vstripes": (x & 1) * 255,
        "hstripes": (y & 1) * 255,
        "diag": ((x - y) % 3 == 0) * 255,
        "flat255": np.full((H, W), 255),
        "hot": np.where((x == 300) & (y == 40), 255, 0),
        "ramp": (x + 3 * y) % 256,
    }
    for name, im in pats.items():
        yield name, im.astype(np.uint8), 32


def main():
    torch.cuda.set_device(0)
    capi.load()
    bad, n = [], 0
    for name, img, rows in images():
        H, W = img.shape
        bands = O.sobel_bands(img, rows)
        in_off, out_off, rws = [], [], []
        pi = po = 0
        for b in bands:
            in_off.append(pi)
            out_off.append(po)
            rws.append(b.shape[0] - 2)
            pi += b.size
            po += (b.shape[0] - 2) * W
        dinp = torch.from_numpy(np.concatenate([b.ravel() for b in bands])).cuda()
        dout = torch.full((po,), 0xA5, dtype=torch.uint8, device="cuda")
        ops.sobel_bands(dinp, in_off, dout, out_off, rws, W)
        want = np.concatenate([O.sobel_band(b, b.shape[0] - 2, W) for b in bands])
        n += 1
        if not np.array_equal(dout.cpu().numpy(), want):
            bad.append(name)
    # claim-pair ring reuse: 2^15 + 3 launches walk the whole self-resetting
    # ring, so the last launches run on slots an earlier launch returned
    img = O.sobel_image(70, 512, 5)
    bands = O.sobel_bands(img, 16)
    dinp = torch.from_numpy(np.concatenate([b.ravel() for b in bands])).cuda()
    in_off = [sum(b.size for b in bands[:i]) for i in range(len(bands))]
    out_off = [sum((b.shape[0] - 2) * 512 for b in bands[:i]) for i in range(len(bands))]
    rws = [b.shape[0] - 2 for b in bands]
    dout = torch.zeros(sum(rws) * 512, dtype=torch.uint8, device="cuda")
    for _ in range((1 << 15) + 3):
        ops.sobel_bands(dinp, in_off, dout, out_off, rws, 512)
    want = np.concatenate([O.sobel_band(b, b.shape[0] - 2, 512) for b in bands])
    n += 1
    if not np.array_equal(dout.cpu().numpy(), want):
        bad.append("ring-reuse")
    env = {k: v for k, v in os.environ.items() if k.startswith("UCG_SOBEL")}
    print(json.dumps({"env": env, "cases": n, "bad": bad}))


if __name__ == "__main__":
    main()
