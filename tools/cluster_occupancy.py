"""cudaOccupancyMaxActiveClusters of the cluster-merge K1 (w4r8 / w8r8) per
cluster size, with the GPU's SM count. usage: python tools/cluster_occupancy.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23798_b200 import _lib  # noqa: E402

h = _lib.lib()
h.elsa_dev_max_active_clusters.restype = ctypes.c_int
h.elsa_dev_max_active_clusters.argtypes = [ctypes.c_int, ctypes.c_int]
torch.cuda.init()
print("SMs:", torch.cuda.get_device_properties(0).multi_processor_count)
for cfg, name in ((0, "w4r8 (2 CTAs/SM)"), (2, "w8r8 (1 CTA/SM)")):
    row = {s: h.elsa_dev_max_active_clusters(cfg, s) for s in (2, 3, 4, 6, 8, 12, 16)}
    print(name, " ".join(f"{s}:{n}({n * s} CTAs)" for s, n in row.items()), flush=True)
