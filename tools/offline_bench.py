"""Time bench.bench_offline alone (POD + DEIM on C2-sized vectors)."""
import json, sys, types
sys.path.insert(0, '.')
import torch, bench
print(json.dumps(bench.bench_offline(types.SimpleNamespace(), torch.device('cuda', 0))))
