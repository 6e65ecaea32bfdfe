import sys, json, types
sys.path.insert(0, '.')
import torch, bench
args = types.SimpleNamespace(warmup=3, steps=12)
for name in sys.argv[1:]:
    print(json.dumps(bench.bench_fom(name, args, torch.device('cuda', 0))))
