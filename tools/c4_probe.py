"""C4 grid-mode docking timings across reduction methods and CTA sizes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2410_10447_b200._lib import load

torch.cuda.set_device(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
print(json.dumps(bench.c4_measure(load(), torch, 0, partitions=tuple(int(x) for x in sys.argv[1:]) or (64, 128, 256)), indent=1))
