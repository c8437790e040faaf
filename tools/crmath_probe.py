import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_10447_b200 import Device
dev = Device(0)
m = np.zeros(8, np.uint64)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
assert dev.lib.mdr_selftest_crmath(dev.ctx, n, m.ctypes.data) == 0
names = ["sin", "cos", "log", "cos2pi"]
print("n", n)
print("correctly rounded vs glibc:", dict(zip(names, m[:4].tolist())))
print("libdevice         vs glibc:", dict(zip(names, m[4:].tolist())))
