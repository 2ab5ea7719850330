"""Run the spectrum loss on a config-2-sized batch (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_01826_b200 import loss
B = 64
S = (torch.randn(B, 360, 180, dtype=torch.complex64, device="cuda") * 0.1)
gt = (S.abs() ** 2 * 1.3 + 0.05).float()
for _ in range(3):
    loss.spectrum_loss_frames(S, gt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    loss.spectrum_loss_frames(S, gt, lam_layout="rays")
e1.record(); torch.cuda.synchronize()
print("loss ms", e0.elapsed_time(e1) / 10)
