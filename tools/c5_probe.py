"""C5 screening sample timing (ligands/hour)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

torch.cuda.set_device(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
print(json.dumps(bench.c5_measure(torch, 0, n_ligands=n), indent=1))
