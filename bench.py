#!/usr/bin/env python
"""bench.py — the CIL hot path (arXiv 2203.14742) on B200.

One step = one pass of the whole hot path over one batch:
  C2 (BASELINE.json configs[1], the headline workload): 100 independent set pairs of
  500 x 500 Gierer-Meinhardt-shaped 64x64x2 patterns, L2, M = 15 radii:
    cil_features (pack -> tcgen05 Gram + fused binning -> exact re-check -> y)
    -> [N > 1: all_gather of the feature vectors over NCCL]
    -> cil_stats (mu_0, Sigma_0 over all vectors) -> cil_loglik (every local vector).
  value = pattern-pair distances per second over all ranks (weak scaling: every rank owns
  100 set pairs).  A secondary line item times C4 (SCIL, Alg. 3, 256 proposals) for the
  "CIL loglik evals/sec" half of the metric.

Launch: python bench.py [--gpus N --steps K --warmup W]  (torchrun for N > 1)
        python bench.py --impl reference ...  -> the FP64 CPU oracle as it stands.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import cilgen  # noqa: E402

METRIC = "pattern-pair distances/sec + CIL loglik evals/sec at 1/2/4/8 B200 vs roofline"
UNIT = "pattern-pair distances/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")

C2 = dict(name="C2", grid=(2, 64, 64), P=100, N=500, Nt=500, M=15, mask=1,
          workload="C2: GM-shaped 64x64x2 patterns, 100 set pairs x (500 x 500), L2, M=15 (BASELINE configs[1])")
C4 = dict(name="C4", grid=(1, 128, 128), P=256, n_ens=10, N_set=50, N_tilde=50, M=13, mask=1,
          workload="C4: SCIL Alg. 3, 256 proposals x pool 1000 of 128x128, n_ens=10, 50+50, L2, M=13")
C6 = dict(name="C6", grid=(2, 64, 64), P=64, N_syn=1000, N_set=50, n_rep=1000, M=13, mask=1,
          workload="C6: SCIL with bootstrapping (Alg. A2), 64 proposals x pool 1000 of 64x64x2, N_set=50, "
                   "n_CIL=1000 replicates, L2, M=13 (PAPER.md:563-564)")
C7 = dict(name="C7", grid=(2, 64, 64), N_set=3000, n_ens=10, M=13, mask=0x3F,
          workload="C7: MCIL-6 training vectors (Alg. 2 steps 1-2) of N_set=3000 GM 64x64x2 patterns, "
                   "n_ens=10 subsets of 300, all six measures, M=13 (PAPER.md:199, 206-226)")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- setup
def launch_ranks(args):
    """--gpus N without a torchrun environment: re-launch this command as N ranks (one process per
    GPU, torch.distributed.run, rendezvous on 127.0.0.1).  Under torchrun, WORLD_SIZE must equal N."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus > 1:
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
            log(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}")
            os.execv(sys.executable, cmd)
    elif int(world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch with matching values")


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def pilot_radii(A0, B0, grid, M):
    """Power-law radii R_m = R_0 b^-m spanning the distances of a 64 x 64
    pilot block: R_0 = max (1 + 1e-3), R_M = min (1 - 1e-3).  Harness setup (untimed)."""
    S, H, W = grid
    h = 1.0 / (W - 1)
    w = h * h if H > 1 else h
    a = A0[:64].reshape(min(64, A0.shape[0]), -1).double()
    b = B0[:64].reshape(min(64, B0.shape[0]), -1).double()
    d = torch.cdist(a, b) * math.sqrt(w)
    d = d[d > 0]
    R0, RM = float(d.max()) * 1.001, float(d.min()) * 0.999
    return R0 * (RM / R0) ** (np.arange(1, M + 1) / M)


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML (the library nvidia-smi
    reads) polled every 20 ms from a thread, each sample time-stamped when taken; nvidia-smi -lms 50
    as the fallback (its piped output arrives in bursts, so short regions get few samples)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvml.h): hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown,
    # sw_power_cap — the order of FIELDS[3:7]
    NVML_BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.nvml = None
        self.stop = False
        self.interval_ms = 50
        self.lines = []                    # (time, csv line)
        self.t0 = self.t1 = None           # the timed region (mark_start / mark_end)

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __enter__(self):
        try:
            uuid = str(torch.cuda.get_device_properties(self.dev).uuid)
            sel = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
        except Exception:
            sel = str(self.dev)
        try:
            import pynvml
            pynvml.nvmlInit()
            h = (pynvml.nvmlDeviceGetHandleByUUID(sel) if sel.startswith("GPU-")
                 else pynvml.nvmlDeviceGetHandleByIndex(int(sel)))
            self.nvml = (pynvml, h)
            self.interval_ms = 20
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", sel, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                flags = ",".join("Active" if rs & b else "Not Active" for b in self.NVML_BITS)
                self.lines.append((time.time(), f"{sm},{mx},{pw:.1f},{flags}"))
            except Exception:
                break
            time.sleep(self.interval_ms / 1000.0)

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi has produced a sample (it takes ~0.1-1 s to start), so a short
        timed region that follows is covered."""
        t_end = time.time() + timeout
        while (self.proc is not None or self.nvml is not None) and not self.lines and time.time() < t_end:
            time.sleep(0.02)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *a):
        self.stop = True
        if self.nvml is not None:
            self.t.join(timeout=1.0)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        """Clocks under load: the samples inside the timed region when there are >= 3 of them (the
        sampler runs from before the warm-up, so a short timed region still has neighbours),
        else every sample from the warm-up start to the end of the timed region."""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [ln for t, ln in self.lines if self.t0 is not None and self.t0 <= t <= (self.t1 or t)]
        window = "timed region" if len(inside) >= 3 else "warm-up + timed region"
        use = inside if len(inside) >= 3 else [ln for t, ln in self.lines if self.t1 is None or t <= self.t1 + 0.06]
        for ln in use:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm), "window": window, "interval_ms": self.interval_ms,
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def timed(fn, steps, stream):
    """CUDA-event time of `steps` calls of fn on `stream` (synchronised both sides), ms."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def engine_used(engine: str, K: int) -> str:
    """The L2 engine AUTO resolves to (include/cil.h): the three-digit INT8 engine (any K)."""
    if engine == "AUTO":
        return "TC_I8"
    return engine


I8_PEAKS_FILE = os.path.join(ROOT, "profiles", "r02_measured_peaks.json")


def tensor_peak(used: str):
    """(dense peak TOP/s, where it comes from, MMA products issued per K element and pair) of the
    engine's tensor-core kind.  int8 / tf32: our own cuBLAS measurement on this pool's B200
    (tools/measure_peaks.py -> profiles/r02_measured_peaks.json, burst); bf16: MEASURED_PEAKS.json."""
    pk = peaks()
    if used == "TC_I8":
        try:
            return (json.load(open(I8_PEAKS_FILE))["int8"]["burst_tops"],
                    "profiles/r02_measured_peaks.json int8 burst (torch._int_mm 8192^3)", 6)
        except Exception:
            return 2.0 * pk.get("bf16_tflops", 1590.0), "MEASURED_PEAKS.json bf16_tflops x 2 (nominal i8:bf16)", 6
    if used == "TC_3XTF32":
        try:
            return (json.load(open(I8_PEAKS_FILE))["tf32"]["burst_tops"],
                    "profiles/r02_measured_peaks.json tf32 burst", 3)
        except Exception:
            return 0.5 * pk.get("bf16_tflops", 1590.0), "MEASURED_PEAKS.json bf16_tflops x 0.5", 3
    return pk.get("bf16_tflops", 1590.0), "MEASURED_PEAKS.json bf16_tflops (burst)", 3


DTYPES = {"TC_I8": "int8 three-digit (22-bit) fixed point / int32 accumulate / f64 stats",
          "TC_3XBF16": "bf16x3 split / f32 accumulate / f64 stats",
          "TC_3XTF32": "tf32x3 split / f32 accumulate / f64 stats",
          "SIMT": "f32 differences / f64 sums"}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def peaks():
    try:
        return json.load(open(PEAKS_FILE))
    except Exception:
        return {}


def traffic_for(key):
    try:
        return json.load(open(TRAFFIC_FILE)).get(key)
    except Exception:
        return None


# --------------------------------------------------------------------------- oracle (CPU)
def oracle_sample_rate(A, B, grid, mask, radii, budget_s=12.0):
    """The FP64 oracle as it stands on the host cores, on whole set pairs of the
    workload (item 0, 1, ...) until ~budget_s of CPU time: returns (pairs/s, cores,
    sample description, seconds)."""
    from oracle import oracle as O
    O.build()
    cores = O.default_threads()
    g = (grid[0], grid[1], grid[2], 0.0)
    pairs, dt, items = 0, 0.0, 0
    while dt < budget_s and items < A.shape[0]:
        a, b = A[items].cpu().numpy(), B[items].cpu().numpy()
        t0 = time.perf_counter()
        O.features(a, b, g, mask, radii, band=0.0, nthreads=cores)
        dt += time.perf_counter() - t0
        pairs += a.shape[0] * b.shape[0]
        items += 1
    return pairs / dt, cores, f"{items} whole set pairs of the workload ({pairs} pairs, L2 counts)", dt


# --------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--engine", default="AUTO", choices=["AUTO", "TC_I8", "TC_3XBF16", "TC_3XTF32", "SIMT"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c6", action="store_true")
    ap.add_argument("--no-c7", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--c5-rows", type=int, default=20000, help="C5 rows per set (BASELINE configs[4]: 20000)")
    ap.add_argument("--c5-mask", type=lambda v: int(v, 0), default=0x3F, help="C5 measures (default all six)")
    ap.add_argument("--c5-steps", type=int, default=2)
    ap.add_argument("--config", default="C2", choices=["C2", "C3"],
                    help="C2 = the headline bench line; C3 = evidence run of the CUDA-core measures")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    launch_ranks(args)

    cfg = C2
    grid, P, N, Nt, M, mask = cfg["grid"], cfg["P"], cfg["N"], cfg["Nt"], cfg["M"], cfg["mask"]
    seed = cilgen.config_seed(2)
    if args.impl == "reference":   # CPU only: rank 0 runs, the other ranks exit 0 without work
        return reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                             cfg, seed, None)

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if args.config == "C3":
        print(json.dumps(bench_c3(args, dev)), flush=True)
        return

    import paper_2203_14742_b200 as cil
    from paper_2203_14742_b200 import _capi

    engine = getattr(cil, "ENGINE_" + args.engine)
    # ---- inputs: each rank owns 100 set pairs (sets 2p, 2p+1 offset by rank), resident in HBM
    t0 = time.time()
    A = torch.empty((P, N) + grid, dtype=torch.float32, device=dev)
    B = torch.empty((P, Nt) + grid, dtype=torch.float32, device=dev)
    for p in range(P):
        q = rank * P + p
        cilgen.make_set(seed, 2 * q, N, grid, device=dev, out=A[p])
        cilgen.make_set(seed, 2 * q + 1, Nt, grid, device=dev, out=B[p])
    # radii from the pilot block of the config's first set pair (identical on every rank)
    A00 = cilgen.make_set(seed, 0, 64, grid, device=dev)
    B00 = cilgen.make_set(seed, 1, 64, grid, device=dev)
    radii_np = pilot_radii(A00, B00, grid, M)
    radii = torch.tensor(radii_np[None, :], dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: generated C2 inputs in {time.time() - t0:.1f}s")

    stream = torch.cuda.current_stream()
    ws = cil.Workspace()
    counts = torch.empty((P, 1, M), dtype=torch.int64, device=dev)
    y = torch.empty((P, 1, M), dtype=torch.float64, device=dev)
    st = torch.empty((P,), dtype=torch.int32, device=dev)
    Yg = torch.empty((world * P, M), dtype=torch.float64, device=dev)
    launches = [0]

    def step():
        cil.features(A, B, grid, mask, radii, engine=engine, ws=ws, counts=counts, y=y, status=st)
        n = cil.last_launch_count()
        if world > 1:
            import torch.distributed as dist
            dist.all_gather_into_tensor(Yg, y.view(P, M))
            Y = Yg
        else:
            Y = y.view(P, M)
        mu, Sig = cil.stats(Y)
        n += cil.last_launch_count()
        out, lst = cil.loglik(mu, Sig, y.view(P, M), ridge=0.0)
        n += cil.last_launch_count()
        launches[0] += n
        return out, lst

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    clk = ClockSampler(local).__enter__().wait_first()   # sampling from before the warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(st.max()) != 0:
        log(f"[bench] WARNING item status {st.unique().tolist()}")

    # ---- timed region (device time, max over ranks)
    launches[0] = 0
    barrier()
    _capi.prof_enable(True)
    clk.mark_start()
    ms = timed(step, args.steps, stream)
    clk.mark_end()
    clk.__exit__()
    _capi.prof_enable(False)
    prof = _capi.prof_read()
    barrier()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    pairs_step = world * P * N * Nt
    value = pairs_step / (ms_step * 1e-3)
    gpu_launches = launches[0]

    # ---- rooflines, live CUDA events around each launch class on its stream (cil_prof_*):
    # the tensor-core Gram (tensor bound) and the INT8 pack (HBM bound); "roofline" is the one
    # with the larger share of the step, the other is reported beside it
    pk = peaks()
    K = grid[0] * grid[1] * grid[2]
    used = engine_used(args.engine, K)
    gram_ms, gram_n = prof["gram_tc"]
    roof_gram = None
    if gram_n > 0:
        per_launch_ms = gram_ms / gram_n
        # split-accounted: the engine issues `nprod` MMA products per K element and pair (INT8: the six
        # digit products hh, hm, mh, hl, mm, lh; float splits: hi.hi + hi.lo + lo.hi)
        peak, psrc, nprod = tensor_peak(used)
        flops = nprod * 2.0 * P * N * Nt * K
        achieved = flops / (per_launch_ms * 1e-3) / 1e12
        kind = {"TC_I8": "INT8 kind::i8, 6 digit products (22-bit fixed point, exact int32)",
                "TC_3XBF16": "3xBF16 kind::f16", "TC_3XTF32": "3xTF32 kind::tf32"}[used]
        roof_gram = {"kernel": "k_gram3 / k_gram_tc: tcgen05 Gram + fused binning, " + kind,
                     "bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 1),
                     "unit": "TOP/s" if used == "TC_I8" else "TFLOP/s",
                     "frac": round(achieved / peak, 4),
                     "peak_source": psrc,
                     "flops_per_launch": flops, "algorithmic_1x_flops_per_launch": flops / nprod,
                     "frac_algorithmic_1x": round(achieved / nprod / peak, 4),
                     "kernel_ms_per_launch": round(per_launch_ms, 4),
                     "kernel_share_of_step": round(gram_ms / ms, 4),
                     "traffic": traffic_for("C2_gram")}
        if used == "TC_I8":
            # the same cuBLAS int8 GEMM run back to back for 4 s (power-capped): the denominator for a
            # kernel that runs inside a long, power-capped step like this one
            try:
                sus = json.load(open(I8_PEAKS_FILE))["int8"]["sustained_tops"]
                roof_gram.update({"peak_sustained": round(sus, 1), "frac_of_sustained": round(achieved / sus, 4),
                                  "peak_sustained_source": "profiles/r02_measured_peaks.json int8 sustained"})
            except Exception:
                pass
    pack_ms, pack_n = prof["pack"]
    roof_pack = None
    if pack_n > 0 and used == "TC_I8":
        # ALGORITHMIC bytes (SURVEY §8(d) per-unit figure: 4K bytes of FP32 read once per
        # pattern) x the patterns of one step; the design additionally writes the three INT8 digit
        # planes (3Kp B per pattern, read back by the Gram) and reads <= 16 centre rows per item —
        # reported separately (achieved_incl_design_bytes), and visible in `traffic` (ncu).
        # Time = the whole pack class (centre + 2 launches).
        Kp = (K + 127) // 128 * 128
        rows = P * (N + Nt)
        nbytes = rows * 4.0 * K
        design_bytes = rows * (4.0 * K + 3.0 * Kp + 32) + P * min(Nt, 16) * 4.0 * K
        sec = pack_ms / args.steps * 1e-3
        achieved = nbytes / sec / 1e9
        hbm = pk.get("hbm_gbs", 6547.0)
        roof_pack = {"kernel": "k_center + 2 x k_pack3: centre, sigma = max|x~|/Q, three INT8 digit planes h, m, l, row metadata",
                     "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)",
                     "algorithmic_bytes_per_step": nbytes,
                     "design_bytes_per_step": design_bytes,
                     "achieved_incl_design_bytes": round(design_bytes / sec / 1e9, 1),
                     "frac_incl_design_bytes": round(design_bytes / sec / 1e9 / hbm, 4),
                     "ms_per_step": round(pack_ms / args.steps, 4),
                     "kernel_share_of_step": round(pack_ms / ms, 4),
                     "traffic": traffic_for("C2_pack")}
    cands = [r for r in (roof_pack, roof_gram) if r is not None]
    roof = max(cands, key=lambda r: r["kernel_share_of_step"]) if cands else None
    roof_other = [r for r in cands if r is not roof]
    kshares = {k: {"ms_per_step": round(v[0] / args.steps, 4), "launches_per_step": v[1] / args.steps}
               for k, v in prof.items() if v[1] > 0}
    listed, _cap = cil.recheck_count(P, N, Nt, grid, mask, M, engine, ws=ws)
    recheck = {"cases_per_step": listed, "fraction_of_pairs": listed / float(P * N * Nt),
               "note": "(pair, measure) cases whose rigorous interval contained a radius -> exact FP64 re-check"}

    # ---- end-to-end through the public API with HOST buffers
    e2e = None
    if not args.no_e2e:
        A_h = torch.empty(A.shape, dtype=torch.float32, pin_memory=True)
        B_h = torch.empty(B.shape, dtype=torch.float32, pin_memory=True)
        A_h.copy_(A)
        B_h.copy_(B)
        out_h = torch.empty((P, 3), dtype=torch.float64, pin_memory=True)
        y_h = torch.empty((P, 1, M), dtype=torch.float64, pin_memory=True)

        # the H2D copy of set-pair chunk c+1 (copy stream) overlaps cil_features of chunk c (the
        # caller's stream); cil_stats / cil_loglik follow once every chunk's y is in
        n_chunks = 4 if P >= 4 else 1
        bounds = [P * c // n_chunks for c in range(n_chunks + 1)]
        cstream = torch.cuda.Stream(device=dev)
        ev_free = torch.cuda.Event()
        ev_in = [torch.cuda.Event() for _ in range(n_chunks)]

        def e2e_step():
            ev_free.record(stream)                     # the previous step's kernels are queued before
            cstream.wait_event(ev_free)
            with torch.cuda.stream(cstream):
                for c in range(n_chunks):
                    c0, c1 = bounds[c], bounds[c + 1]
                    A[c0:c1].copy_(A_h[c0:c1], non_blocking=True)
                    B[c0:c1].copy_(B_h[c0:c1], non_blocking=True)
                    ev_in[c].record(cstream)
            for c in range(n_chunks):
                c0, c1 = bounds[c], bounds[c + 1]
                stream.wait_event(ev_in[c])
                cil.features(A[c0:c1], B[c0:c1], grid, mask, radii, engine=engine, ws=ws,
                             counts=counts[c0:c1], y=y[c0:c1], status=st[c0:c1])
            Y = y.view(P, M)
            if world > 1:
                import torch.distributed as dist
                dist.all_gather_into_tensor(Yg, Y)
                Y = Yg
            mu, Sig = cil.stats(Y)
            out, _ = cil.loglik(mu, Sig, y.view(P, M), ridge=0.0)
            out_h.copy_(out, non_blocking=True)
            y_h.copy_(y, non_blocking=True)

        y_dev = y.clone()                              # y of the device-resident step
        e2e_step()
        barrier()
        e_ms = timed(e2e_step, args.e2e_steps, stream)
        e2e_same = bool(torch.equal(y, y_dev))         # chunked host path reproduces it exactly
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item()) / args.e2e_steps
        e2e = {"value": pairs_step / (e_ms * 1e-3), "unit": UNIT, "ms_per_step": round(e_ms, 3),
               "h2d_bytes_per_step": int(A.nbytes + B.nbytes), "d2h_bytes_per_step": int(out_h.nbytes + y_h.nbytes),
               "steps": args.e2e_steps, "h2d_chunks_overlapped": n_chunks, "y_equals_device_step": e2e_same}
        del A_h, B_h

    # ---- secondary: C4 (SCIL) loglik evals/s
    c4 = None
    if not args.no_c4:
        c4 = bench_c4(cil, args, world, rank, dev, engine, stream)
    c6 = None
    if not args.no_c6:
        c6 = bench_c6(cil, args, world, rank, dev, engine, stream)
    c7 = None
    if not args.no_c7:
        c7 = bench_c7(cil, args, world, rank, dev, engine, stream)
    # ---- CPU baseline: the oracle as it stands, bounded sample, rank 0 at N = 1 only
    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        rate, cores, sample, dt = oracle_sample_rate(A, B, grid, mask, radii_np[None, :])
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
               "seconds": round(dt, 2), "cpu_model": cpu_model()}
    c3 = None
    if not args.no_c3:
        c3 = bench_c3(args, dev)
    c5 = None
    if not args.no_c5:
        del A, B
        torch.cuda.empty_cache()
        c5 = bench_c5(cil, args, world, rank, dev, engine, stream)


    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPES[engine_used(args.engine, grid[0] * grid[1] * grid[2])],
            "data": "synthetic (cilgen-v1 seeded generator, resident in HBM)",
            "config": {"workload": cfg["workload"], "set_pairs_per_gpu": P, "N": N, "Nt": Nt,
                       "grid_SHW": list(grid), "M": M, "measures": ["L2"], "engine": args.engine,
                       "parallelism": f"set pairs sharded over {world} GPU(s), all_gather of y over NCCL"
                       if world > 1 else "1 GPU",
                       "l2_flush": "inputs (3.28 GB per GPU) exceed the 126 MB L2; no explicit flush",
                       "radii": [float(r) for r in radii_np]},
            "loglik_evals_per_s": world * P / (ms_step * 1e-3),
            "clocks": clk.summary(),
            "gpu_launches": gpu_launches,
            "roofline": roof,
            "roofline_other": roof_other[0] if roof_other else None,
            "kernel_breakdown": kshares,
            "recheck": recheck,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "secondary": c4,
            "secondary_bootstrap": c6,
            "secondary_train": c7,
            "secondary_c3": c3,
            "secondary_c5": c5,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def pilot_radii_all(A0, B0, grid, M, mask):
    """Harness radii for every selected measure from a 64 x 64 pilot block (torch, untimed,
    harness setup only): power law between max (1 + 1e-3) and min (1 - 1e-3)."""
    S, H, W = grid
    h = 1.0 / (W - 1)
    w = h * h if H > 1 else h
    a = A0[:64].double()
    rows = []
    for i in range(a.shape[0]):
        u = a[i:i + 1] - B0[:64].double()                      # [64, S, H, W]
        dx = torch.diff(u, dim=-1) / h
        dy = torch.diff(u, dim=-2) / h
        a0 = (w * (u ** 2).flatten(1).sum(1)).sqrt()
        ax = (w * (dx ** 2).flatten(1).sum(1)).sqrt()
        ay = (w * (dy ** 2).flatten(1).sum(1)).sqrt() if H > 1 else torch.zeros_like(a0)
        m0 = u.abs().flatten(1).amax(1)
        mx = dx.abs().flatten(1).amax(1)
        my = dy.abs().flatten(1).amax(1) if H > 1 else torch.zeros_like(m0)
        rows.append(torch.stack([a0, m0, a0 + ax + ay, (a0 ** 2 + ax ** 2 + ay ** 2).sqrt(),
                                 torch.maximum(m0, torch.maximum(mx, my)), m0 + mx + my]))
    d = torch.cat(rows, dim=1)                                 # [6, 64*64]
    out = []
    for q in range(6):
        if (mask >> q) & 1:
            R0, RM = float(d[q].max()) * 1.001, float(d[q].min()) * 0.999
            out.append(R0 * (RM / R0) ** (np.arange(1, M + 1) / M))
    return np.array(out)


def bench_c5(cil, args, world, rank, dev, engine, stream):
    """C5 (BASELINE configs[4]): ONE large cross-set pair, N = Nt = 20000 patterns of 256x256x2,
    L2 + the alternative measures (default all six), M = 20, the pair space row-block sharded over
    the ranks (north star): rank r takes A rows row_range(N, G, r) against all of B
    (sharding.sharded_features) and the int64 count vectors are all-reduced over NCCL — the only
    exchange.  Strong scaling (total work fixed).  The counts are printed so runs at different G can
    be compared: integer sums are order-free and every rank's engines see the same B, so they must
    be bit-identical for every G."""
    import hashlib

    import torch.distributed as dist

    from paper_2203_14742_b200 import _capi, sharding
    grid, M, mask = (2, 256, 256), 20, args.c5_mask
    N = Nt = args.c5_rows
    seed = cilgen.config_seed(5)
    lo, hi = sharding.row_range(N, world, rank)
    K = grid[0] * grid[1] * grid[2]
    nq = bin(mask).count("1")
    need_ws = cil.features_workspace_size(1, hi - lo, Nt, grid, mask, M, engine)
    need = need_ws + 4 * K * ((hi - lo) + Nt)
    free = torch.cuda.mem_get_info(dev)[0]
    res = {"workload": f"C5: one cross-set pair of {N} x {Nt} GM 256x256x2 patterns, measures mask {mask:#x}, M={M}, "
                       f"rows sharded over {world} GPU(s), NCCL all_reduce of the int64 counts (BASELINE configs[4])",
           "metric": "pattern-pair distances/s (all measures of the mask per pair)", "scaling": "strong",
           "rows_this_rank": [lo, hi], "bytes_needed_per_rank": need, "bytes_free": free}
    flag = torch.tensor([1 if need < 0.92 * free else 0], dtype=torch.int32, device=dev)
    if world > 1:
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 0:
        res["skipped"] = "insufficient device memory on some rank"
        return res
    t0 = time.time()
    A = cilgen.make_set(seed, 0, hi - lo, grid, device=dev, row0=lo)
    B = cilgen.make_set(seed, 1, Nt, grid, device=dev)
    P0a = cilgen.make_set(seed, 0, 64, grid, device=dev)
    radii = torch.tensor(pilot_radii_all(P0a, B[:64], grid, M, mask), dtype=torch.float64, device=dev)
    del P0a
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: generated C5 rows [{lo}, {hi}) + B ({Nt}) in {time.time() - t0:.1f}s")
    ws = cil.Workspace()

    last = [None]

    def step():
        last[0] = sharding.sharded_features(A, B, grid, mask, radii, N, engine=engine, ws=ws)
        return last[0]

    clk = ClockSampler(dev.index or 0).__enter__().wait_first()
    step()                                               # warm-up (kernel attributes, workspace)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    _capi.prof_enable(True)
    steps = max(1, args.c5_steps)
    clk.mark_start()
    ms = timed(step, steps, stream)
    clk.mark_end()
    clk.__exit__()
    _capi.prof_enable(False)
    prof = _capi.prof_read()
    if world > 1:
        dist.barrier()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / steps
    counts, y, st = last[0]
    torch.cuda.synchronize()
    listed, cap = cil.recheck_count(1, hi - lo, Nt, grid, mask, M, engine, ws=ws)
    c = counts[0].cpu().numpy().astype(np.int64)
    pk_i8, psrc, nprod = tensor_peak("TC_I8")
    kb = {k: round(v[0] / steps, 3) for k, v in prof.items() if v[1] > 0}
    res.update({"value": N * Nt / (ms_step * 1e-3), "ms_per_step": round(ms_step, 2), "steps": steps, "warmup": 1,
                "item_status": int(st[0].item()),
                "counts": c.tolist(), "counts_sha256": hashlib.sha256(c.tobytes()).hexdigest()[:16],
                "clocks_this_rank": clk.summary(),
                "recheck_cases_this_rank": listed, "recheck_fraction_this_rank": listed / float((hi - lo) * Nt * nq),
                "kernel_breakdown_this_rank": kb})
    if prof["gram_tc"][1]:
        g_ms = prof["gram_tc"][0] / steps
        S_, H_, W_ = grid
        Kaug = K + S_ * H_ * (W_ - 1) + S_ * (H_ - 1) * W_ if mask & 0x0C else K
        ops = nprod * 2.0 * (hi - lo) * Nt * Kaug
        res["gram_tc_this_rank"] = {"ms": round(g_ms, 2), "achieved_tops": round(ops / (g_ms * 1e-3) / 1e12, 1),
                                    "peak": round(pk_i8, 1), "peak_source": psrc,
                                    "frac": round(ops / (g_ms * 1e-3) / 1e12 / pk_i8, 4)}
    del A, B, ws
    torch.cuda.empty_cache()
    return res


def bench_c3(args, dev):
    """Evidence run for SURVEY §8 config C3 (the alternative measures): 2000 x 2000 patterns of
    128x128x2, all six measures, M = 20.  AUTO: L2, W12, W12SUM on the three-phase INT8 tensor-core
    engine, the max family (Linf, W1inf, W1infsum) on the CUDA-core engine; SIMT: everything on
    CUDA cores."""
    import paper_2203_14742_b200 as cil
    from paper_2203_14742_b200 import _capi
    grid, N, M, mask = (2, 128, 128), 2000, 20, 0x3F
    seed = cilgen.config_seed(3)
    A = cilgen.make_set(seed, 0, N, grid, device=dev)
    B = cilgen.make_set(seed, 1, N, grid, device=dev)
    radii = torch.tensor(pilot_radii_all(A, B, grid, M, mask), dtype=torch.float64, device=dev)
    engine = getattr(cil, "ENGINE_" + args.engine)
    ws = cil.Workspace()
    stream = torch.cuda.current_stream()

    def step():
        cil.features(A, B, grid, mask, radii, engine=engine, ws=ws)

    clk = ClockSampler(dev.index or 0).__enter__().wait_first()   # sampling from before the warm-up
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 20))                  # >= 0.4 s timed: >= 8 clock samples at 50 ms
    _capi.prof_enable(True)
    clk.mark_start()
    ms = timed(step, steps, stream) / steps
    clk.mark_end()
    _capi.prof_enable(False)
    clk.__exit__()
    prof = _capi.prof_read()
    S, H, W = grid
    K = S * H * W
    Kaug = K + S * H * (W - 1) + S * (H - 1) * W
    simt_ms = prof["simt_tile"][0] / max(1, prof["simt_tile"][1])
    ep = float(N) * N * Kaug                                  # element-pairs per family per launch
    tc_family = args.engine in ("AUTO", "TC_I8")
    # AUTO / TC_I8: the max family alone on the 15-bit fixed-point engine (max16.cu: IMAD +
    # VIMNMX3.U16x2); SIMT: both families on the FP32 engine (FADD2 + FMNMX3 + FFMA2)
    mix = 3 if tc_family else 0
    ceil, _ = _capi.alu_ceiling(mix)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    # pipe ceiling of the fixed-point mix: VIMNMX3.U16x2 issues at 16 lanes / SMSP / cycle on the
    # integer pipe and covers 2 element-pairs per lane -> 128 element-pairs per SM-cycle (the IMADs
    # go to the FMA pipe at the same rate), at the maximum SM clock
    pipe_ceil = 128.0 * nsm * 1965e6 if tc_family else None
    res = {"workload": "C3: 2000 x 2000 of 128x128x2, all six measures, M=20",
           "engine": args.engine,
           "ms_per_step": round(ms, 3), "pairs_per_s": N * N / (ms * 1e-3),
           "simt_tile": {"families": "max (Linf, W1inf, W1infsum)" if tc_family else "max + L2-type",
                         "ms_per_launch": round(simt_ms, 3), "element_pairs_per_s": ep / (simt_ms * 1e-3),
                         "alu_ceiling_element_pairs_per_s": ceil,
                         "ceiling_mix": "IMAD+VIMNMX3.U16x2 (measured, register-only)" if mix == 3
                         else "FADD2+FMNMX3+FFMA2 (measured, register-only)",
                         "frac": round(ep / (simt_ms * 1e-3) / ceil, 4), "K_aug": Kaug,
                         "pipe_ceiling_element_pairs_per_s": pipe_ceil,
                         "frac_of_pipe_ceiling": round(ep / (simt_ms * 1e-3) / pipe_ceil, 4) if pipe_ceil else None},
           "kernel_breakdown": {k: round(v[0] / steps, 3) for k, v in prof.items() if v[1] > 0},
           "clocks": clk.summary()}
    g_ms, g_n = prof["gram_tc"]
    if g_n and tc_family:
        per = g_ms / g_n
        peak, psrc, nprod = tensor_peak("TC_I8")
        ops = nprod * 2.0 * N * N * Kaug                     # three-phase Gram over [x | D_x x | D_y x]
        ach = ops / (per * 1e-3) / 1e12
        res["gram_tc"] = {"engine": "TC_I8 three-phase (L2, W12, W12SUM)", "ms_per_launch": round(per, 3),
                          "achieved_tops": round(ach, 1), "peak": round(peak, 1), "peak_source": psrc,
                          "frac_of_peak": round(ach / peak, 4)}
    listed, _ = cil.recheck_count(1, N, N, grid, mask, M, engine, ws=ws)
    res["recheck"] = {"cases_per_step": listed, "fraction_of_pair_measures": listed / (6.0 * N * N)}
    res["metric"] = "pattern-pair distances/s (all six measures per pair)"
    res["value"] = N * N / (ms * 1e-3)
    del A, B, ws
    torch.cuda.empty_cache()
    return res


def bench_c6(cil, args, world, rank, dev, engine, stream):
    """Secondary line for the bootstrap row: Alg. A2 loglik evals/s at the
    paper's sizes (N_syn = 1000, n_CIL = 1000 replicates), L2, per-theta
    radii; draws seeded on the host (untimed inputs, like the patterns)."""
    cfg = C6
    grid, P, N_syn, N_set, n_rep, M = cfg["grid"], cfg["P"], cfg["N_syn"], cfg["N_set"], cfg["n_rep"], cfg["M"]
    seed = cilgen.config_seed(6)
    t0 = time.time()
    pools = torch.empty((P, N_syn) + grid, dtype=torch.float32, device=dev)
    for p in range(P):
        u = cilgen.uniforms(seed, 5000 + rank * P + p, np.array([0]), 2)[0]
        cilgen.make_set(seed, rank * P + p, N_syn, grid, device=dev, out=pools[p], n_w=4.5 + u[0],
                        amp_scale=0.8 + 0.4 * u[1])
    data = cilgen.make_set(seed, 100000, N_set, grid, device=dev)
    draws = [cilgen.boot_draws_a2(seed, rank * P + p, n_rep, N_syn, N_set) for p in range(P)]
    I1 = torch.tensor(np.stack([d[0] for d in draws]), device=dev)
    I2 = torch.tensor(np.stack([d[1] for d in draws]), device=dev)
    J = torch.tensor(np.stack([d[2] for d in draws]), device=dev)
    radii = torch.tensor(np.stack([pilot_radii(pools[p, :64], pools[p, 64:128], grid, M)[None, :] for p in range(P)]),
                         dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: generated C6 pools + draws in {time.time() - t0:.1f}s")
    ws = cil.Workspace()
    out = torch.empty((P, 3), dtype=torch.float64, device=dev)
    st = torch.empty((P,), dtype=torch.int32, device=dev)

    def step():
        cil.synth_loglik_boot(pools, data, N_set, I1, I2, J, grid, cfg["mask"], radii, ridge=1e-10, engine=engine,
                              ws=ws, out=out, status=st)

    clk = ClockSampler(dev.index or 0).__enter__().wait_first()
    for _ in range(args.warmup):
        step()
    steps = max(3, args.steps // 40)
    from paper_2203_14742_b200 import _capi
    _capi.prof_enable(True)
    clk.mark_start()
    ms = timed(step, steps, stream)
    clk.mark_end()
    clk.__exit__()
    _capi.prof_enable(False)
    prof = _capi.prof_read()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / steps
    K = grid[0] * grid[1] * grid[2]
    Nt = N_syn - N_set
    res = {"workload": cfg["workload"], "metric": "SCIL-bootstrap loglik evals/s", "value": world * P / (ms_step * 1e-3),
           "ms_per_step": round(ms_step, 3), "steps": steps,
           "pool_pairs_per_s": world * P * N_syn * N_syn / (ms_step * 1e-3),
           "resampled_pairs_per_s": world * P * n_rep * N_set * Nt / (ms_step * 1e-3),
           "nonzero_status": int((st != 0).sum())}
    g_ms, g_n = prof["gram_tc"]
    if g_n:
        per_step = g_ms / steps
        # both Gram launches of a step: the pool x pool bin matrix and the y~ counts (s_data x pool[J])
        used = engine_used(args.engine, K)
        peak, psrc, nprod = tensor_peak(used)
        # issued: the pool x pool bin matrix runs the tile upper triangle (256 x 128 tiles, tile row mt
        # from column tile 2 mt on), the y~ leg one 64-column tile per 256 pool rows; unique: the
        # N_syn (N_syn + 1) / 2 pool pairs + the N_set x N_syn y~ pairs the method needs
        tm, tn = -(-N_syn // 256), -(-N_syn // 128)
        issued = P * (sum(tn - 2 * m for m in range(tm)) * 256 * 128 + tm * 256 * 64)
        unique = P * (N_syn * (N_syn + 1) / 2 + N_set * N_syn)
        t_s = per_step * 1e-3
        res["gram_tc"] = {"engine": used, "ms_per_step": round(per_step, 4), "launches_per_step": g_n / steps,
                          "achieved_tops_issued": round(nprod * 2.0 * issued * K / t_s / 1e12, 1),
                          "frac_of_peak_issued": round(nprod * 2.0 * issued * K / t_s / 1e12 / peak, 4),
                          "achieved_tops_unique_pairs": round(nprod * 2.0 * unique * K / t_s / 1e12, 1),
                          "frac_of_peak_unique_pairs": round(nprod * 2.0 * unique * K / t_s / 1e12 / peak, 4),
                          "peak": round(peak, 1), "peak_source": psrc}
    r_ms, r_n = prof["resample"]
    if r_n:
        # steps 2.1-2.4: multiplicities, 0/1 threshold rows E, one integer GEMM (rows M1 of the
        # replicates x rows of E, K = N_syn) whose epilogue applies the column multiplicities.
        # Algorithmic int8 ops of the GEMM: 2 n_rep (M N_syn) N_syn per item.
        r_step = r_ms / steps
        res["resample"] = {"ms_per_step": round(r_step, 4), "launches_per_step": r_n / steps,
                           "engine": "tc_rowdot" if engine != cil.ENGINE_SIMT and N_set <= 127 else "atoms",
                           "lookups_per_s": P * n_rep * N_set * Nt / (r_step * 1e-3),
                           "gemm_int8_tops_incl_helpers": round(2.0 * P * n_rep * M * N_syn * N_syn / (r_step * 1e-3)
                                                                / 1e12, 1)}
    res["kernel_breakdown"] = {k: round(v[0] / steps, 4) for k, v in prof.items() if v[1] > 0}
    res["clocks"] = clk.summary()
    return res


def bench_c7(cil, args, world, rank, dev, engine, stream):
    """Secondary line for the Alg. 1 / Alg. 2 training row: the C(n_ens, 2)
    subset-pair vectors of one large data set, all six measures (L2-type family on the
    tensor cores, max family on the CUDA cores, k >= l tiles skipped)."""
    cfg = C7
    grid, N_set, n_ens, M, mask = cfg["grid"], cfg["N_set"], cfg["n_ens"], cfg["M"], cfg["mask"]
    seed = cilgen.config_seed(7)
    X = cilgen.make_set(seed, rank, N_set, grid, device=dev)
    N = N_set // n_ens
    radii = torch.tensor(pilot_radii_all(X[:N], X[N:2 * N], grid, M, mask), dtype=torch.float64, device=dev)
    ws = cil.Workspace()

    def step():
        cil.train_vectors(X, n_ens, grid, mask, radii, engine=engine, ws=ws)

    clk = ClockSampler(dev.index or 0).__enter__().wait_first()
    for _ in range(max(2, args.warmup)):
        step()
    steps = max(3, args.steps // 80)
    from paper_2203_14742_b200 import _capi
    _capi.prof_enable(True)
    clk.mark_start()
    ms = timed(step, steps, stream)
    clk.mark_end()
    clk.__exit__()
    _capi.prof_enable(False)
    prof = _capi.prof_read()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / steps
    nv = n_ens * (n_ens - 1) // 2
    res = {"workload": cfg["workload"], "metric": "training vectors/s", "value": world * nv / (ms_step * 1e-3),
           "ms_per_step": round(ms_step, 3), "steps": steps,
           "pairs_per_s": world * nv * N * N / (ms_step * 1e-3),
           "kernel_breakdown": {k: round(v[0] / steps, 4) for k, v in prof.items() if v[1] > 0}}
    g_ms, g_n = prof["gram_tc"]
    if g_n:
        S_, H_, W_ = grid
        Kaug = S_ * H_ * W_ + S_ * H_ * (W_ - 1) + S_ * (H_ - 1) * W_
        peak, psrc, nprod = tensor_peak("TC_I8")
        per = g_ms / g_n
        ops = nprod * 2.0 * nv * N * N * Kaug                # the k < l blocks the method needs
        res["gram_tc"] = {"engine": "TC_I8 three-phase (L2, W12, W12SUM), k < l tiles only",
                          "ms_per_launch": round(per, 3), "achieved_tops_on_needed_pairs": round(ops / (per * 1e-3) / 1e12, 1),
                          "peak": round(peak, 1), "peak_source": psrc,
                          "frac_of_peak_on_needed_pairs": round(ops / (per * 1e-3) / 1e12 / peak, 4)}
    res["clocks"] = clk.summary()
    return res


def bench_c4(cil, args, world, rank, dev, engine, stream):
    cfg = C4
    grid, P, n_ens, N_set, Nt, M = cfg["grid"], cfg["P"], cfg["n_ens"], cfg["N_set"], cfg["N_tilde"], cfg["M"]
    seed = cilgen.config_seed(4)
    Nsyn = n_ens * (N_set + Nt)
    t0 = time.time()
    pools = torch.empty((P, Nsyn) + grid, dtype=torch.float32, device=dev)
    rng = np.random.default_rng(seed + rank)
    for p in range(P):
        # theta-dependence emulated by the wavelength count and amplitude
        u = cilgen.uniforms(seed, 5000 + rank * P + p, np.array([0]), 2)[0]
        cilgen.make_set(seed, rank * P + p, Nsyn, grid, device=dev, out=pools[p], n_w=4.5 + u[0], amp_scale=0.8 + 0.4 * u[1])
    data = cilgen.make_set(seed, 1000, N_set, grid, device=dev)
    k0 = torch.tensor([p % n_ens for p in range(P)], dtype=torch.int32, device=dev)
    radii = torch.tensor(np.stack([pilot_radii(pools[p, :64], pools[p, 64:128], grid, M)[None, :] for p in range(P)]),
                         dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: generated C4 pools in {time.time() - t0:.1f}s")
    ws = cil.Workspace()
    out = torch.empty((P, 3), dtype=torch.float64, device=dev)
    st = torch.empty((P,), dtype=torch.int32, device=dev)

    def step():
        cil.synth_loglik(pools, n_ens, N_set, Nt, data, k0, grid, cfg["mask"], radii, ridge=1e-10, engine=engine,
                         ws=ws, out=out, status=st)

    clk = ClockSampler(dev.index or 0).__enter__().wait_first()
    for _ in range(args.warmup):
        step()
    steps = max(3, args.steps // 10)
    from paper_2203_14742_b200 import _capi
    _capi.prof_enable(True)
    clk.mark_start()
    ms = timed(step, steps, stream)
    clk.mark_end()
    clk.__exit__()
    _capi.prof_enable(False)
    prof = _capi.prof_read()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / steps
    K = grid[0] * grid[1] * grid[2]
    rowsA, rowsB = (n_ens + 1) * N_set, n_ens * Nt
    g_ms, g_n = prof["gram_tc"]
    res = {"workload": cfg["workload"], "metric": "CIL loglik evals/s", "value": world * P / (ms_step * 1e-3),
           "ms_per_step": round(ms_step, 3), "steps": steps,
           "pairs_per_s": world * P * rowsA * rowsB / (ms_step * 1e-3),
           "nonzero_status": int((st != 0).sum())}
    if g_n:
        per = g_ms / g_n
        used = engine_used(args.engine, K)
        peak, psrc, nprod = tensor_peak(used)
        ach = nprod * 2.0 * P * rowsA * rowsB * K / (per * 1e-3) / 1e12
        res["gram_tc"] = {"engine": used, "ms_per_launch": round(per, 4), "achieved_tops": round(ach, 1),
                          "peak": round(peak, 1), "peak_source": psrc, "frac_of_peak": round(ach / peak, 4)}
    res["kernel_breakdown"] = {k: round(v[0] / steps, 4) for k, v in prof.items() if v[1] > 0}
    res["clocks"] = clk.summary()
    return res


def reference_arm(args, world, rank, cfg, seed, dev):
    """--impl reference: the FP64 oracle as it stands on the host cores (this tier's
    reference arm), same metric/config; each step a bounded sample of the workload."""
    if rank != 0:
        return
    grid, N, Nt, M, mask = cfg["grid"], cfg["N"], cfg["Nt"], cfg["M"], cfg["mask"]
    from oracle import oracle as O
    O.build()
    A0 = cilgen.make_set(seed, 0, N, grid)
    B0 = cilgen.make_set(seed, 1, Nt, grid)
    radii = pilot_radii(A0, B0, grid, M)[None, :]
    cores = O.default_threads()
    a, b = A0.numpy(), B0.numpy()
    g = (grid[0], grid[1], grid[2], 0.0)
    rows = cores  # one row per core per step: bounded (~seconds) sample of the workload
    t0 = time.perf_counter()
    O.features(a[:rows], b, g, mask, radii, band=0.0, nthreads=cores)
    per = time.perf_counter() - t0
    total_budget = 150.0
    steps, warm = args.steps, args.warmup
    if (steps + warm) * per > total_budget:
        steps = max(1, int(total_budget / per) - warm)
    for _ in range(warm):
        O.features(a[:rows], b, g, mask, radii, band=0.0, nthreads=cores)
    t0 = time.perf_counter()
    for s in range(steps):
        r0 = (s * rows) % (N - rows + 1)
        O.features(a[r0:r0 + rows], b, g, mask, radii, band=0.0, nthreads=cores)
    dt = time.perf_counter() - t0
    value = steps * rows * Nt / dt
    sample = f"{rows} rows x all {Nt} of set pair 0 per step (L2 counts, FP64 oracle)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": round(dt / steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (cilgen-v1)",
            "config": {"workload": cfg["workload"], "grid_SHW": list(grid), "M": M, "measures": ["L2"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
