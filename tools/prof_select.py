"""Run the selector alone (cfg3 shape) a few times; used under ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_15197_b200 import ops  # noqa: E402

B, k, C = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 16, 8192
g = torch.Generator(device="cuda").manual_seed(0)
conf = (torch.rand(B, k, dtype=torch.float64, device="cuda", generator=g) ** 0.3).contiguous()
for _ in range(6):
    ops.select(conf, C)
torch.cuda.synchronize()
