"""Decode alone (ResNet-50 shapes, rho = 0.001): P emulated ranks' messages decoded on one GPU,
mu = 0 (latency) and mu = 0.9 (GB/s against 16 d + 8 pairs).  Prints one JSON line per P."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ks_for, measure_decode, resnet50_dims  # noqa: E402

dims = resnet50_dims()
ks = ks_for(dims)
for P in [int(x) for x in (sys.argv[1:] or ["2", "4", "8"])]:
    print(json.dumps(measure_decode(dims, ks, torch.device("cuda", 0), P=P)), flush=True)
