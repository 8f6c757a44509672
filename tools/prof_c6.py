"""Run the C6 bootstrap evaluation (Alg. A2) a few times, for ncu captures of its kernels.
usage: python tools/prof_c6.py [reps]"""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2203_14742_b200 as cil

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
args = types.SimpleNamespace(warmup=1, steps=3 * 40, engine="AUTO")
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream()
res = bench.bench_c6(cil, args, 1, 0, dev, cil.ENGINE_AUTO, stream)
print({k: res[k] for k in ("ms_per_step", "resample", "nonzero_status")})
