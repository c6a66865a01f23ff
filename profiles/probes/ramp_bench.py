"""Times the FDK ramp-filter stage on config 2's raw line integrals (496 x
1248 x 960) on the device: the fused kernel (default) or cuFFT
(CBB_RAMP_CUFFT=1). Prints ms per stack and the HBM rate on 8 B/pixel."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.num_projections
torch.manual_seed(0)
raw = torch.randn((n, cfg.height, cfg.width), device="cuda", dtype=torch.float32)
out = torch.empty_like(raw)
pkg.ramp_filter_device(raw, out, cfg.pixel_mm)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
a.record()
for _ in range(reps):
    pkg.ramp_filter_device(raw, out, cfg.pixel_mm)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
px = raw.numel()
impl = "cufft" if os.environ.get("CBB_RAMP_CUFFT") else "fused"
print(f"{impl} {cfg.name} {n}x{cfg.height}x{cfg.width}: {ms:.3f} ms per stack, "
      f"{8 * px / ms / 1e6:.1f} GB/s on 8 B/pixel, {px / 2 / ms / 1e3:.0f} k row-pairs/ms")
