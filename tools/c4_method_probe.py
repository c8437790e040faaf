"""One C4 grid docking with a given reduction method (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2410_10447_b200._lib import load

torch.cuda.set_device(0)
torch.cuda.set_stream(torch.cuda.Stream())
m = sys.argv[1]
part = int(sys.argv[2]) if len(sys.argv) > 2 else 128
print(bench.c4_measure(load(), torch, 0, methods=(m,), partitions=(part,), steps=1)["results"])
