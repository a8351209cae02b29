"""Per-stage norm-relative error of the reference harness's whole-network
gradients (tests/refharness) for alternative builds of libscc_b200.so
(LD_LIBRARY_PATH overrides the in-tree library)."""
import json, os, subprocess, sys
import numpy as np
B = "tests/refharness/_build"
def grad(exe, env=None, model="mobilenet_like.json", batch=4, spatial=32):
    o = subprocess.run([f"{B}/{exe}", f"{B}/models/{model}", "grad", str(batch), str(spatial)], capture_output=True, text=True, env=env, timeout=600)
    assert o.returncode == 0, o.stderr
    return json.loads(o.stdout)
def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
for model, batch, sp in (("mobilenet_like.json", 4, 32), ("two_block.json", 8, 8)):
    r = grad("train_ref", model=model, batch=batch, spatial=sp)
    for tag in sys.argv[1:]:
        env = dict(os.environ)
        if tag != "current":
            env["LD_LIBRARY_PATH"] = os.path.abspath(tag) + ":" + env.get("LD_LIBRARY_PATH", "")
        g = grad("train_b200", env, model=model, batch=batch, spatial=sp)
        errs = [round(nrel(sg["weight"], sr["weight"]), 7) for sg, sr in zip(g["stages"], r["stages"])]
        print(model, tag, "logits", f"{nrel(g['logits'], r['logits']):.2e}", "stage dW", errs, "head", f"{nrel(g['head_weight'], r['head_weight']):.2e}", flush=True)
