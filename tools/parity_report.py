"""Print the parity reports (image and gradient errors vs the reference's golden
fixtures) for the small full fixtures and the full-size summaries."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from conftest import load_golden  # noqa: E402
from parity import grad_report, image_report  # noqa: E402
from test_gpu_parity import FULL_FIXTURES, run_gpu  # noqa: E402

from paper_2406_02720_b200 import scenes  # noqa: E402

out = {}
for name, (gen, kernel) in FULL_FIXTURES.items():
    gold = load_golden(name)
    got = run_gpu(gen(), int(gold["cam_idx"]), kernel, torch.float32,
                  gold["d_color"] if "d_color" in gold else None)
    ref = {k: gold[k] for k in ("color", "alpha", "depth", "transmittance", "terminal")}
    rep = image_report(got, ref)
    if "d_mu" in gold:
        rep["grads"] = grad_report(got, {k: gold[k] for k in gold if k.startswith("d_") or
                                         k == "pos_grad_norm"})
    out[name] = rep
print(json.dumps(out, indent=1, default=float))
