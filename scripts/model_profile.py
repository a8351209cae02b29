"""One eager SCC-ResNet-18 training step (batch 128) for an ncu launch list:
  ncu --metrics gpu__time_duration.sum --csv python scripts/model_profile.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_00745_b200.models import MODELS
torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
m = MODELS[name](device="cuda")
opt = torch.optim.SGD(m.parameters(), lr=0.05, momentum=0.9)
x = torch.randn(128, 3, 32, 32, device="cuda"); y = torch.randint(0, 10, (128,), device="cuda")
for _ in range(3):
    opt.zero_grad(); torch.nn.functional.cross_entropy(m(x), y).backward(); opt.step()
torch.cuda.synchronize()
