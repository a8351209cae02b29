"""SCC-ResNet-18 / SCC-VGG16 (CIFAR shape, batch 128) and SCC-ResNet-50
(ImageNet shape, batch 256) synthetic training images/sec on one GPU (or under
torchrun: data parallel over NCCL, per-GPU batch fixed)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2101_00745_b200.train import train_throughput
ws = int(os.environ.get("WORLD_SIZE", "1"))
if ws > 1:
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl")
else:
    torch.cuda.set_device(0)
RUNS = {"resnet18": dict(batch=128, steps=20, warmup=5), "vgg16": dict(batch=128, steps=20, warmup=5),
        "resnet50": dict(batch=256, steps=8, warmup=3, image=224, num_classes=1000)}
for name in (sys.argv[1:] or ["resnet18", "vgg16", "resnet50"]):
    r = train_throughput(name, **RUNS[name])
    if ws == 1 or dist.get_rank() == 0:
        print(json.dumps(r), flush=True)
if ws > 1:
    dist.destroy_process_group()
