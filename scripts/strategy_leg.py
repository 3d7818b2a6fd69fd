"""The bench's weight-policy comparison leg alone (bench_pipeline.strategy_comparison)."""
import json, sys, torch
sys.path.insert(0, '.')
from paper_2312_00839_b200 import bench_pipeline as bp
print(json.dumps(bp.strategy_comparison(torch, torch.device('cuda', 0))))
