import sys, os, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2101_00745_b200 as scc
from fp64_ref import scc_fp64
for mode in (0, 1):
  os.environ.pop('SCC_FWD_R32', None)
  if mode: os.environ['SCC_FWD_R32'] = '1'
  for (n, h, w) in ((2, 8, 8), (1, 8, 8), (2, 16, 16), (32, 32, 32)):
      cfg = scc.scc_config_new(64, 128, 2, "50%", True)
      cfg.set_path(scc._lib.SCC_PATH_TENSOR)
      torch.manual_seed(0)
      x = torch.randn(n, 64, h, w, device="cuda")
      wts = scc.scc_weights_init(cfg)
      y = scc.scc_forward(x, wts, cfg)
      torch.cuda.synchronize()
      dy = torch.zeros(n, 128, h, w, device="cuda")
      r = scc_fp64(64, 128, 32, 16, x, wts.weight, wts.bias, dy)
      ry = r[0].reshape(n, 128, h, w).cpu().numpy()
      d = np.abs(y.cpu().numpy() - ry)
      bad = np.argwhere(d > 1e-3)
      print(mode, (n, h, w), "bad", len(bad), "of", d.size, "samples", np.unique(bad[:, 0])[:8] if len(bad) else None,
            "chan", np.unique(bad[:, 1])[:8] if len(bad) else None, flush=True)
