"""Where does the device densify differ from the reference fixture? (diagnostic)"""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
import adam_cases as A  # noqa: E402
from conftest import load_golden  # noqa: E402
from test_gpu_densify import _setup  # noqa: E402
from paper_2406_02720_b200 import trainer as T  # noqa: E402

gold = load_golden("densify")
for name in gold["cases"]:
    c = A.densify_case(gold, name)
    scene, stats, opt, cfg = _setup(c, torch.float64)
    new, _, rep = T.densify_and_prune(scene, stats, cfg, opt, np.random.default_rng(c["seed"]),
                                      c["extent"])
    nk = c["out"]["mu"].shape[0] - rep["cloned"] - 2 * rep["split"]
    for f in ("mu", "log_scale"):
        got = getattr(new, f).cpu().numpy()
        ref = c["out"][f]
        bad = np.nonzero(np.any(got != ref, axis=1))[0]
        ulps = np.abs(got - ref) / np.spacing(np.abs(ref))
        print(name, f, "kept", nk, "clones", rep["cloned"], "bad rows", bad[:10], len(bad),
              "max ulps", ulps.max())
