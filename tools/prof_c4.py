"""Run the C4 SCIL evaluation (Alg. 3) a few times, for ncu captures of its kernels.
usage: python tools/prof_c4.py"""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2203_14742_b200 as cil

args = types.SimpleNamespace(warmup=1, steps=3 * 40, engine="AUTO")
res = bench.bench_c4(cil, args, 1, 0, torch.device("cuda:0"), cil.ENGINE_AUTO, torch.cuda.current_stream())
print({k: res.get(k) for k in ("value", "ms_per_step", "kernel_breakdown")})
