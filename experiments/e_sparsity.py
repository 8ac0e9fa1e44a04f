"""Fraction of 32x32 E tiles (and cells) that are exactly zero in fp32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_17206_b200 import Engine
eng = Engine(0)
for name, (B, L, D, g) in {"c1": (4, 256, 128, 1.0), "c2": (4, 1024, 128, 0.1), "c3": (2, 4096, 128, 0.01),
                           "c4": (4, 256, 1024, 1.0), "c2g1": (4, 1024, 128, 1.0), "bary": (4, 512, 64, 1.0)}.items():
    gen = torch.Generator(device="cuda").manual_seed(1)
    if name == "bary":
        t = torch.linspace(0, 1, L, device="cuda")
        x = (torch.sin(6 * t)[None, :, None] + 0.05 * torch.randn((B, L, D), generator=gen, device="cuda"))
        y = (torch.sin(6 * t + 0.5)[None, :, None] + 0.05 * torch.randn((B, L, D), generator=gen, device="cuda"))
    else:
        x = torch.randn((B, L, D), generator=gen, device="cuda"); y = torch.randn((B, L, D), generator=gen, device="cuda")
    loss, E = eng.forward_backward_E(x.contiguous(), y.contiguous(), g)
    E = E[:, 1:-1, 1:-1].float()
    nz = (E != 0)
    tiles = nz.reshape(B, L // 32, 32, L // 32, 32).any(dim=4).any(dim=2)
    big = (E > 1e-7)
    tb = big.reshape(B, L // 32, 32, L // 32, 32).any(dim=4).any(dim=2)
    print(f"{name}: nonzero cells {nz.float().mean().item():.4f}  nonzero tiles {tiles.float().mean().item():.4f}  tiles with E>1e-7 {tb.float().mean().item():.4f}")
