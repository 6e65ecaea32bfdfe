"""One FOM RK2-average step on a config's mesh (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import types
import numpy as np
import torch
import bench
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
args = types.SimpleNamespace(warmup=2, steps=4)
print(bench.bench_fom(name, args, torch.device('cuda', 0)))
