"""One eager SCC-ResNet-18 training step (batch 128) for an ncu launch list:
  ncu --metrics gpu__time_duration.sum --csv python scripts/model_profile.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_00745_b200.models import MODELS
torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
big = name == "resnet50"
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
m = MODELS[name](device="cuda", num_classes=1000 if big else 10)
opt = torch.optim.SGD(m.parameters(), lr=0.05, momentum=0.9)
b, hw = (256, 224) if big else (128, 32)
x = torch.randn(b, 3, hw, hw, device="cuda"); y = torch.randint(0, 1000 if big else 10, (b,), device="cuda")
for _ in range(3):
    opt.zero_grad(); torch.nn.functional.cross_entropy(m(x), y).backward(); opt.step()
torch.cuda.synchronize()
