"""Raw scoring throughput (bench.score_throughput)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2410_10447_b200._lib import load

torch.cuda.set_device(0)
torch.cuda.set_stream(torch.cuda.Stream())
print(json.dumps(bench.score_throughput(load(), torch, 0), indent=1))
