"""Write GPU-produced attention outputs as ATN1 candidate files for the
reference's own verifier: `scanattn verify --candidate`
(cli.py:155-165) and `verify.bound_check(candidate=...)` (verify.py:320-335)
consume them in tests/test_reference_verify_cpu.py.

Run on a GPU box:  python tools/make_gpu_candidates.py
Inputs are the reference generator's problems (oracle.generate, pinned
bitwise to scanattn.generate by tests/golden/generator.npz); every output is
computed by libelsa's FP32 forward through the public drop-in.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2604_23798_b200 as elsa  # noqa: E402
from paper_2604_23798_b200 import tensorio  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "gpu_candidates")

# (name, scenario, seed, dims b,h,n,d,dv) — presets of tensorio.py:118-122 and
# the acceptance problems of test_acceptance.py:56-57, 169-171, plus d = 64
CASES = [
    ("regular_preset", "regular", 11, (2, 4, 256, 32, 32)),
    ("long_preset", "long", 11, (1, 1, 4096, 32, 32)),
    ("stress_preset", "stress", 11, (2, 2, 1024, 32, 32)),
    ("accept_n256", "regular", 11, (1, 1, 256, 16, 8)),
    ("accept_n1024", "regular", 11, (1, 1, 1024, 16, 8)),
    ("accept_n4096", "regular", 11, (1, 1, 4096, 16, 8)),
    ("regular_d64", "regular", 0, (1, 2, 1024, 64, 64)),
    ("long_d64", "long", 0, (1, 1, 4096, 64, 64)),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    dev = torch.device("cuda", 0)
    manifest = []
    for name, scen, seed, (b, h, n, d, dv) in CASES:
        Q, K, V = oracle.generate(seed, scen, b=b, h=h, n=n, d=d, d_v=dv, dtype=np.float32)
        q, k, v = (torch.from_numpy(x).to(dev) for x in (Q, K, V))
        y = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
        torch.cuda.synchronize()
        path = os.path.join(OUT, name + ".atn")
        tensorio.write_tensor(path, y)
        manifest.append({"name": name, "scenario": scen, "seed": seed,
                         "dims": [b, h, n, d, dv], "plan": elsa.describe_plan(q, k, v),
                         "device": torch.cuda.get_device_name(dev)})
        print(name, manifest[-1]["plan"], flush=True)
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
