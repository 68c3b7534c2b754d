"""Device time of the fused image loss (cs_image_loss) at the config-5 view
size: python tools/loss_timing.py [H W]"""
import sys

import torch

from paper_2411_14974_b200 import train_ops

H, W = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (840, 1297)
g = torch.Generator(device="cuda").manual_seed(0)
img = torch.rand((H, W, 3), generator=g, device="cuda")
tgt = torch.rand((H, W, 3), generator=g, device="cuda")
masks = torch.randn(1_000_000, generator=g, device="cuda")
dm = torch.zeros_like(masks)
lw = train_ops.LossWorkspace()
for _ in range(3):
    train_ops.image_loss(img, tgt, masks, 0.2, 5e-4, d_raw_mask=dm, workspace=lw)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    train_ops.image_loss(img, tgt, masks, 0.2, 5e-4, d_raw_mask=dm, workspace=lw)
e1.record()
torch.cuda.synchronize()
print(f"image_loss {H}x{W}: {e0.elapsed_time(e1) / 20 * 1000:.1f} us per call")
