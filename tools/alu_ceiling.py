import sys, os; sys.path.insert(0, os.getcwd())
from paper_2203_14742_b200 import _capi
import torch
for m in (3, 1, 0):
    for _ in range(2): v, ms = _capi.alu_ceiling(m)
    print(m, v, v / 148 / 1.965e9, "per SM-cycle at 1965 MHz", ms)
