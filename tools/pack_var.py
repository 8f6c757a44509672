"""Times the C4 pack (and step) for one build of libcil.so: python tools/pack_var.py TAG
(tools/simt_var.sh-style A/B of pack variants; prints one line)."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_14742_b200 as cil  # noqa: E402

args = types.SimpleNamespace(warmup=3, steps=20 * 10, engine="AUTO")
res = bench.bench_c4(cil, args, 1, 0, torch.device("cuda:0"), cil.ENGINE_AUTO, torch.cuda.current_stream())
kb = res["kernel_breakdown"]
print(f"{sys.argv[1] if len(sys.argv) > 1 else '-':24s} C4 step {res['ms_per_step']:.3f} ms  pack {kb['pack']:.3f}  "
      f"gram {kb['gram_tc']:.3f}  status {res['nonzero_status']}  clocks {res['clocks'].get('sm_mhz')}")
