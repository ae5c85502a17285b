#!/usr/bin/env python
"""bench.py -- SecONNds server-side HE-linear-layer time on B200 (BASELINE.json metric).

A step is one pass of the whole hot path over every conv layer of SqueezeNet 1.1 at 224x224
(BASELINE.json configs[2]) with the paper's 37-bit BFV parameters
(N = 4096, Q = q0 q1 of 60 + 49 bits, t = 2^37; reading R1): per layer the
server-share add + forward NTT of the input ciphertexts, the NTT-domain ct x pt MAC against the
NTT-preprocessed weights, the inverse NTT + random mask, and the extraction of the server's
output share -- all in libsecn's sm_100a kernels through its C ABI. Inputs are synthetic and
seeded (workloads/inputs.py); they are resident in HBM before the timed region (2.9 GB per
step, far larger than the 126 MB L2, so no explicit flush is needed).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl secn|reference]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ...  (output-channel sharding, NCCL
all-gather of the server's output shares; time = max over ranks).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from workloads import inputs, layers  # noqa: E402

METRIC = "SqueezeNet HE-linear-layer time (s)"
NET_INFO = {  # --net -> (metric, BASELINE.json config index, description)
    "squeezenet1_1": (METRIC, 2, "all 26 conv layers of SqueezeNet 1.1 at 224x224"),
    "squeezenet1_0": (METRIC, 2, "all 26 conv layers of SqueezeNet 1.0 at 224x224"),
    "resnet50": ("ResNet-50 HE-linear-layer time (s)", 3, "all 53 conv layers of ResNet-50 v1.5 at 224x224"),
    "tiny": ("tiny HE conv time (s)", 0, "single 3x3 conv, 16x16x4 -> 8 channels"),
}


def net_info(net):
    m, i, desc = NET_INFO.get(net, (METRIC, 2, net))
    return m, f"{net}: {desc} (BASELINE.json configs[{i}])"
HBM_PEAK_FALLBACK = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["secn", "reference"], default="secn")
    ap.add_argument("--net", default="squeezenet1_1",
                    help="squeezenet1_1 (C3, default) | squeezenet1_0 | resnet50 (C4) | tiny (C1) | ntt_sweep (C5)")
    ap.add_argument("--word-bits", type=int, choices=[32, 64], default=32,
                    help="32: four 27-bit uint32 RNS limbs (reading R1b, headline); 64: q 60+49 bit uint64 limbs "
                         "(reading R1)")
    ap.add_argument("--no-companion", action="store_true",
                    help="skip the timing-only run of the other word size reported under 'companion'")
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--cpu-frac", type=float, default=None,
                    help="fraction of every layer's output ciphertexts the oracle computes (default 1 = the whole "
                         "network, measured; ResNet-50 0.02, extrapolated)")
    ap.add_argument("--mask", choices=["device", "host"], default="device",
                    help="device (default): the server's mask r is drawn inside every layer call (secn32_he_conv2d_gen, "
                         "Philox4x32-10, reading R17); host: r is a caller input (secn32_he_conv2d_ex)")
    ap.add_argument("--mask-schedule", choices=["ahead", "lookahead", "inline"], default="ahead",
                    help="device mask: when each layer's mask is drawn + encoded (secn_mask_encode) -- ahead "
                         "(default): every layer's at the start of the step, on a side stream beside the layer chain "
                         "(1.209 ms, profiles/r02h_*); lookahead: the next group's while a group runs (1.253 ms); "
                         "inline: inside the layer call, secn32_he_conv2d_gen (1.232 ms)")
    ap.add_argument("--priority", choices=["chain", "same"], default="chain",
                    help="chain: the layer chain's streams at high priority, the mask side stream at the "
                         "default (the scheduler prefers the latency-bound chain's CTAs); same: all default")
    ap.add_argument("--queries", type=int, default=1,
                    help="B > 1: the batched-queries line instead -- B independent inferences per step (the "
                         "north star's ciphertext batches), each on its own stream, weights shared; metric = "
                         "inferences/s over all ranks (weak scaling: every rank runs its own B)")
    ap.add_argument("--batched-leg", type=int, default=8,
                    help="queries of the batched leg reported under 'batched_queries' in the default run (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-online", action="store_true", help="skip the online-NTT-preprocessing (f4) leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the compact NTT sweep (C5) in the default run")
    ap.add_argument("--overlap", choices=["none", "staged", "free"], default="free",
                    help="layers reading the same input (fire e1/e3, ResNet c1/ds): free (default) = whole layers "
                         "on side streams; staged = the group's layers run each launch group (NTT, MAC, tail) side "
                         "by side and join between groups; none = network order on one stream")
    ap.add_argument("--concurrent", action="store_const", const="free", dest="overlap",
                    help="alias of --overlap free")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", HBM_PEAK_FALLBACK)), "measured"
    return HBM_PEAK_FALLBACK, "fallback"


# ------------------------------------------------------------------------------------------
# clocks during the timed region (NVML)

class ClockSampler:
    """Samples SM clocks and clock-event reasons with `nvidia-smi -lms` in a separate process for
    the duration of the timed region (the B200_PROFILING.md clocks line)."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period_ms: int = 20):
        self.index, self.period_ms = index, period_ms
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._p = None

    def __enter__(self):
        import subprocess

        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.05)
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            return
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 3:
                continue
            try:
                sm, mx, bits = float(f[0]), float(f[1]), int(f[2], 16)
            except ValueError:
                continue
            self.max_mhz = mx
            if bits & ~0x1:  # ignore samples where only gpu_idle is set (between launches)
                for b, name in self.REASONS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            self.samples.append(sm)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "sampler": "nvidia-smi -lms 20"}


# ------------------------------------------------------------------------------------------
# workload

def mask_seed(seed):
    """The bench's Philox key for the device-drawn mask (reading R17); the stream id is the layer index."""
    return (0x5EC0_11D5_0000_0000 ^ (seed * 0x9E3779B97F4A7C15)) & (2**64 - 1)


def layer_inputs(P_primes, n, t_bits, lay, opl_G, opl_S, M, seed):
    """Seeded synthetic inputs of one layer (identical on every rank and in the oracle)."""
    g = inputs.rng(seed)
    ct = inputs.uniform_residues(g, (opl_G * opl_S, 2), P_primes, n)
    x0 = inputs.uniform_below(g, (opl_G * opl_S, n), 1 << t_bits)
    K = inputs.quantized_kernel(g, M, lay.C, lay.k, lay.k, t_bits)
    r = inputs.uniform_below(g, (M * opl_S, n), 1 << t_bits)
    return ct, x0, K, r


def algorithmic_bytes(plan, L, n, wbytes=8, drawn_mask=False):
    """SURVEY.md §8d per-layer bytes: wb L N (2GS + MG + 2MS) + 8 N MS (+ 8 N GS for x0; + 8 N MS
    more when the mask is drawn on the device: the draw writes r, the tail reads it)."""
    G, S, M = plan.G, plan.S, plan.M
    return (wbytes * L * n * (2 * G * S + M * G + 2 * M * S) + 8 * n * M * S + 8 * n * G * S
            + (8 * n * M * S if drawn_mask else 0))


def stage_bytes(plan, L, n, wbytes=8):
    """Bytes each launch group reads + writes (its own roofline numerator)."""
    G, S, M = plan.G, plan.S, plan.M
    ct_in = 2 * G * S * L * n * wbytes
    x0 = G * S * n * 8
    w = M * G * L * n * wbytes
    y = 2 * M * S * L * n * wbytes
    r = M * S * n * 8
    return {0: ct_in + x0 + ct_in, 1: w + ct_in + y, 2: y + r + y}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl" if args.impl == "secn" else "gloo")
    if args.impl == "reference":
        return run_reference(args, world, rank)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import __graft_entry__

    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    if args.net == "ntt_sweep":
        return run_ntt_sweep_line(args, world, rank, local, dev)
    if args.queries > 1:
        return run_batched_line(args, world, rank, local, dev)
    out = run_secn(args, args.word_bits, world, rank, local, dev, full=True)
    if args.batched_leg > 1:
        torch.cuda.empty_cache()
        bq = run_batched(args, args.batched_leg, world, rank, local, dev)
        if rank == 0:
            out["batched_queries"] = bq
    if not args.no_sweep:
        torch.cuda.empty_cache()
        sw = ntt_sweep(args, world, local, dev, word_bits=(args.word_bits,), steps=10)
        if rank == 0:
            out["ntt_sweep"] = sw
    if not args.no_companion:
        other = 64 if args.word_bits == 32 else 32
        torch.cuda.empty_cache()
        comp = run_secn(args, other, world, rank, local, dev, full=False)
        if rank == 0:
            out["companion"] = comp
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_batched(args, B, world, rank, local, dev):
    """B independent inferences of the network per step (the ciphertext-batch axis): query b has
    its own seeded inputs, device-drawn masks (stream id 1000 b + layer) and outputs and runs the
    whole layer chain on its own stream; the weights are preprocessed once and shared. Captured as
    one CUDA graph; device time with CUDA events (max over ranks; every rank runs its own B)."""
    from paper_2506_11586_b200 import Context, MaskGen

    ctx = Context(local, word_bits=args.word_bits)
    L, n = ctx.L, ctx.n
    net = layers.network(args.net)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
    R = ((lambda a: T(a)) if ctx.word_bits == 64 else
         (lambda a: torch.from_numpy(np.ascontiguousarray(a).astype(np.uint32).view(np.int32)).to(dev)))
    lay_state = []
    for li, lay in enumerate(net):
        plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
        g = inputs.rng(args.seed * 1000 + li)
        w = ctx.preprocess_weights(plan, T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k, ctx.t_bits)))
        qs = []
        for b in range(B):
            gq = inputs.rng(10_000_000 + 1000 * (rank * B + b) + li)
            qs.append({"ct": R(inputs.uniform_residues(gq, (plan.G * plan.S, 2), ctx.primes, n)),
                       "x0": T(inputs.uniform_below(gq, (plan.G * plan.S, n), 1 << ctx.t_bits)),
                       "gen": MaskGen(seed=mask_seed(args.seed), stream=1000 * (rank * B + b) + li, ct0=0),
                       "em": ctx.empty(plan.M * plan.S, L, n), "out": ctx.empty(plan.M * plan.S, 2, L, n),
                       "y0": torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=dev),
                       "ws": torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev)})
        lay_state.append((plan, w, qs))
    streams = [torch.cuda.Stream(dev) for _ in range(B)]

    def step():
        main = torch.cuda.current_stream(dev)
        for b, s in enumerate(streams):
            s.wait_stream(main)
            with torch.cuda.stream(s):
                for plan, w, qs in lay_state:
                    q = qs[b]
                    ctx.mask_encode(plan, gen=q["gen"], out=q["em"], y0=q["y0"])
                for plan, w, qs in lay_state:
                    q = qs[b]
                    ctx.he_conv2d_em(plan, q["ct"], w, q["em"], x0=q["x0"], out=q["out"], workspace=q["ws"])
        for s in streams:
            main.wait_stream(s)

    ms = graph_ms(step, args.steps, max(args.warmup, 3), dev, world)
    # the B concurrent streams against one query at a time: queries 0 and B-1 re-run eagerly on
    # one stream into fresh buffers must give the graph's words (ciphertexts and shares) exactly
    torch.cuda.synchronize()
    compared = mismatched = 0
    for b in sorted({0, B - 1}):
        for plan, w, qs in lay_state:
            q = qs[b]
            em, y0 = ctx.empty(plan.M * plan.S, L, n), torch.empty_like(q["y0"])
            ctx.mask_encode(plan, gen=q["gen"], out=em, y0=y0)
            out = ctx.he_conv2d_em(plan, q["ct"], w, em, x0=q["x0"], workspace=q["ws"])
            torch.cuda.synchronize()
            mismatched += int((out != q["out"]).sum().item()) + int((y0 != q["y0"]).sum().item())
            compared += out.numel() + y0.numel()
    total = B * world
    alg = sum(algorithmic_bytes(plan, L, n, ctx.word_bits // 8, True) for plan, _, _ in lay_state) * B
    ctx.close()
    return {"queries_per_gpu": B, "value": round(total / (ms / 1e3), 1), "unit": "inferences/s",
            "ms_per_step": round(ms, 4), "latency_per_query_ms_upper": round(ms, 4),
            "hbm_frac": round(alg / (ms / 1e3) / 1e9 / peaks()[0], 4),
            "graph_vs_eager": {"queries_checked": sorted({0, B - 1}), "words_compared": compared,
                               "words_mismatched": mismatched},
            "path": "per query: secn_mask_encode (drawn masks) then secn32_he_conv2d_em for every layer, on the "
                    "query's own stream; B streams concurrently, weights shared"}


def run_batched_line(args, world, rank, local, dev):
    with ClockSampler(local) as clk:
        bq = run_batched(args, args.queries, world, rank, local, dev)
    if rank == 0:
        out = {"metric": f"{args.net} HE-linear-layer throughput (inferences/s)", "value": bq["value"],
               "unit": "inferences/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": bq["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": f"u{args.word_bits}", "data": "synthetic",
               "config": {"workload": net_info(args.net)[1] + f", {args.queries} independent queries per GPU",
                          "parallelism": f"query batches: {args.queries} per rank, no collective",
                          "timing": "CUDA events around CUDA-graph replays (max over ranks)"},
               "batched_queries": bq, "gpu_launches": None, "clocks": clk.summary()}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


SWEEP_PRIMES = {64: (0xFFFFFFFFFFC0001, 0xFFFFFFFFF840001, 0xFFFFFFFFF6A0001, 0xFFFFFFFFF5A0001),
                32: (0x7E90001, 0x7E00001, 0x7DD0001, 0x7D70001)}  # = 1 mod 2^16: every N <= 2^15


def ntt_sweep(args, world, local, dev, word_bits=(32, 64), steps=20, logns=(12, 13, 14, 15), limbs=(1, 2, 3, 4)):
    """batched RNS NTT / INTT over N = 2^12..2^15 and 1..4 limbs, each call on
    a batch of >= 1 GiB of uniform residues (independent batches per rank). Device time per call
    from CUDA-graph replays (max over ranks); NTT/s counts limb-poly transforms (all ranks)."""
    from paper_2506_11586_b200 import Context

    hbm_peak, _ = peaks()
    gib = 1 << 30
    buf = torch.empty(gib // 8, dtype=torch.int64, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    rows = []
    for wb in word_bits:
        wbytes = wb // 8
        for logn in logns:
            for L in limbs:
                primes = SWEEP_PRIMES[wb][:L]
                ctx = Context(local, log_n=logn, primes=primes, word_bits=wb)
                n = 1 << logn
                n_polys = max(1, gib // (n * wbytes * L))
                words = n_polys * L * n
                t = buf.view(torch.int32 if wb == 32 else torch.int64)[:words].view(n_polys, L, n)
                t.random_(0, min(primes), generator=g)
                res = {"word_bits": wb, "N": n, "L": L, "limb_polys": n_polys * L}
                for name, fn in (("fwd", ctx.ntt_fwd), ("inv", ctx.ntt_inv)):
                    ms = graph_ms(lambda: fn(t), steps, 3, dev, world)
                    res[name + "_us"] = round(ms * 1e3, 2)
                    res[name + "_ntt_per_s"] = round(n_polys * L * world / (ms / 1e3), 1)
                    gbps = 2 * words * wbytes / (ms / 1e3) / 1e9
                    res[name + "_hbm_frac"] = round(gbps / hbm_peak, 4)
                rows.append(res)
                ctx.close()
    del buf
    torch.cuda.empty_cache()
    return rows


def run_ntt_sweep_line(args, world, rank, local, dev):
    """`--net ntt_sweep`: the C5 configuration as its own bench line. value = forward NTT/s at
    N = 4096 with four 27-bit limbs (all ranks); the full grid is under "sweep"."""
    if rank == 0:
        import __graft_entry__  # noqa: F401  (built by main)
    with ClockSampler(local) as clk:
        rows = ntt_sweep(args, world, local, dev, word_bits=(32, 64), steps=args.steps)
    head = next(r for r in rows if r["word_bits"] == args.word_bits and r["N"] == 4096 and r["L"] == (4 if args.word_bits == 32 else 2))
    if rank == 0:
        out = {"metric": "batched RNS NTT throughput (limb-poly transforms/s)", "value": head["fwd_ntt_per_s"],
               "unit": "NTT/s", "n_gpus": world, "steps": args.steps, "warmup": 3,
               "ms_per_step": round(head["fwd_us"] / 1e3, 4), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": f"u{args.word_bits}", "data": "synthetic uniform residues",
               "config": {"workload": "ntt_sweep: N=2^12..2^15 x L=1..4, >= 1 GiB per call (BASELINE.json configs[4])",
                          "headline": f"N=4096, L={head['L']}, {args.word_bits}-bit limbs, forward",
                          "l2": "1 GiB per call >> 126 MB L2"},
               "roofline": {"bound": "hbm", "achieved": round(head["fwd_hbm_frac"] * peaks()[0], 1), "peak": peaks()[0],
                            "unit": "GB/s", "frac": head["fwd_hbm_frac"], "traffic": None},
               "gpu_launches": args.steps, "clocks": clk.summary(), "sweep": rows}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_secn(args, word_bits, world, rank, local, dev, full):
    """Builds the workload at one residue word size, times K graph replays of the step and (full)
    the per-stage, e2e and cpu_baseline legs. Returns the JSON dict on rank 0 (None elsewhere)."""
    from paper_2506_11586_b200 import Context, MaskGen
    from paper_2506_11586_b200 import dist as sdist
    from paper_2506_11586_b200.schedule import GroupRunner, StagedGroupRunner, concurrent_groups

    ctx = Context(local, word_bits=word_bits)
    drawn = args.mask == "device"
    L, n, t_bits = ctx.L, ctx.n, ctx.t_bits
    wbytes = ctx.word_bits // 8

    def R(a):  # residues -> device tensor of the context's word size
        a = np.ascontiguousarray(a)
        return torch.from_numpy(a.view(np.int64) if wbytes == 8 else a.astype(np.uint32).view(np.int32)).to(dev)
    net = layers.network(args.net)

    # ---- setup: plans, inputs, offline weight preprocessing (timed separately) ----
    st = []
    for li, lay in enumerate(net):
        plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
        parts = sdist.partition(plan.M, plan.S, world)  # (channel x spatial-block) rectangle per rank
        m0, mc = parts[rank].m0, parts[rank].mc
        ct, x0, K, r = layer_inputs(ctx.primes, n, t_bits, lay, plan.G, plan.S, plan.M, args.seed * 1000 + li)
        S = plan.S
        d = {"lay": lay, "plan": plan, "win": (plan.Hw, plan.Ww, plan.decim == 2), "m0": m0, "mc": mc, "ct_h": ct, "x0_h": x0,
             "K_h": K, "r_h": r, "parts": parts}
        if mc > 0:
            sl = parts[rank].sc < plan.S  # a spatial slice: only these blocks' output cts (include/secn.h)
            pl = plan.copy(M=mc, s_begin=parts[rank].s0 if sl else 0, s_count=parts[rank].sc if sl else 0)
            d["pl"] = pl
            d["ct"] = R(ct)
            d["x0"] = torch.from_numpy(x0.view(np.int64)).to(dev)
            d["K"] = torch.from_numpy(np.ascontiguousarray(K[m0:m0 + mc]).view(np.int64)).to(dev)
            if drawn:  # this rank's rows of the layer's mask (ct0 = m0 S); r itself only for the stage legs
                d["gen"] = MaskGen(seed=mask_seed(args.seed), stream=li, ct0=m0 * S)
                d["r"] = ctx.mask_draw(d["gen"], mc * S)
                d["ws_gen"] = torch.empty((ctx.gen_workspace_bytes(pl) + 7) // 8, dtype=torch.int64, device=dev)
                d["em"] = ctx.empty(mc * S, L, n)  # the encoded mask (secn_mask_encode), for the side-stream schedules
            else:
                d["r"] = torch.from_numpy(np.ascontiguousarray(r[m0 * S:(m0 + mc) * S]).view(np.int64)).to(dev)
            d["out"] = ctx.empty(mc * S, 2, L, n)
            d["ws"] = torch.empty(ctx.workspace_bytes(pl) // 8, dtype=torch.int64, device=dev)
        else:
            d["pl"] = None
        st.append(d)
    dims = [(d["plan"].M, d["plan"].OH, d["plan"].OW) for d in st]
    layout = sdist.share_layout(dims, world, [d["parts"] for d in st])
    share_buf = torch.zeros(layout.chunk, dtype=torch.int64, device=dev)
    for d, off in zip(st, layout.offsets):
        if d["mc"] > 0:
            d["y0"] = share_buf[off:off + d["mc"] * d["plan"].OH * d["plan"].OW].view(d["mc"], d["plan"].OH, d["plan"].OW)

    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for d in st:
        if d["mc"] > 0:
            d["w"] = ctx.preprocess_weights(d["pl"], d["K"])
    e1.record()
    torch.cuda.synchronize()
    offline_s = e0.elapsed_time(e1) / 1e3

    # layers that read the same input tensor (fire e1/e3, ResNet c1/ds) overlap on side streams;
    # everything else keeps network order (paper_2506_11586_b200/schedule.py)
    names = [d["lay"].name for d in st]
    groups = concurrent_groups(names) if args.overlap != "none" else [[i] for i in range(len(st))]
    hi = -1 if args.priority == "chain" else 0  # torch maps it to the device's highest priority
    runner = StagedGroupRunner(groups, dev) if args.overlap == "staged" else GroupRunner(groups, dev, priority=hi)

    # device mask drawn + encoded apart from the layer call (it is input-independent): on a side
    # stream, ahead of the layer that adds it; the layer's stream waits for its event
    msched = args.mask_schedule if drawn and args.overlap != "staged" else "inline"
    mstream = torch.cuda.Stream(dev)
    mev = [torch.cuda.Event() for _ in st]

    def encode_mask(i):
        d = st[i]
        if d["mc"] > 0:
            with torch.cuda.stream(mstream):
                ctx.mask_encode(d["pl"], gen=d["gen"], out=d["em"], y0=d["y0"])
                mev[i].record(mstream)

    def layer_call(i):
        d = st[i]
        if d["mc"] > 0 and drawn and msched != "inline":
            torch.cuda.current_stream().wait_event(mev[i])  # recorded before this layer was issued
            ctx.he_conv2d_em(d["pl"], d["ct"], d["w"], d["em"], x0=d["x0"], out=d["out"], workspace=d["ws"])
        elif d["mc"] > 0 and drawn:
            ctx.he_conv2d_gen(d["pl"], d["ct"], d["w"], d["gen"], x0=d["x0"], out=d["out"], workspace=d["ws_gen"],
                              y0=d["y0"])
        elif d["mc"] > 0:
            ctx.he_conv2d(d["pl"], d["ct"], d["w"], x0=d["x0"], r=d["r"], out=d["out"], workspace=d["ws"],
                          y0=d["y0"])

    def stage_call(i, k):
        d = st[i]
        if d["mc"] > 0:
            ctx.he_conv2d_stage_ex(k, d["pl"], d["ct"], d["w"], d["x0"], d["r"], d["out"], d["y0"], d["ws"])

    def before_group(k):  # lookahead: group k+1's masks on the side stream while group k runs
        if k + 1 < len(runner.groups):
            mstream.wait_stream(torch.cuda.current_stream())
            for i in runner.groups[k + 1]:
                encode_mask(i)

    def step_public():
        ahead = drawn and msched != "inline"
        if ahead:
            mstream.wait_stream(torch.cuda.current_stream())
            for i in (range(len(st)) if msched == "ahead" else runner.groups[0]):
                encode_mask(i)
        if args.overlap == "staged":
            runner(layer_call, stage_call)
        else:
            runner(layer_call, before_group if ahead and msched == "lookahead" else None)
        if ahead:
            torch.cuda.current_stream().wait_stream(mstream)

    # ---- warmup (eager), then capture the step in a CUDA graph ----
    for _ in range(max(args.warmup, 3)):
        step_public()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev, priority=hi)
    cap.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cap):
        step_public()
    torch.cuda.current_stream(dev).wait_stream(cap)
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=cap):
        step_public()
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        graph.replay()
        sdist.all_gather_shares(share_buf, world)
    torch.cuda.synchronize()

    # ---- timed region: K graph replays (+ the share all-gather when N > 1) ----
    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for i in range(K):
            evs[i][0].record()
            graph.replay()
            gathered = sdist.all_gather_shares(share_buf, world)
            evs[i][1].record()
        torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(total_ms.item()) / K

    if world > 1 and rank == 0:
        shares = sdist.reassemble(gathered, layout, dims, world, [d["parts"] for d in st],
                                  [sdist.block_of_output(d["plan"]) for d in st])
        assert all(f.shape[0] == M for f, (M, _, _) in zip(shares, dims))
    hbm_peak, peak_kind = peaks()
    alg_bytes = sum(algorithmic_bytes(d["plan"], L, n, wbytes, drawn) for d in st)
    step_s = ms_per_step / 1e3
    if not full:
        del graph
        stage_ms = stage_profile(ctx, st, K, dev)  # every rank runs the eager stage calls together
        if rank != 0:
            return None
        return {"dtype": f"u{ctx.word_bits}", "primes": [hex(q) for q in ctx.primes], "limbs": L,
                "value": round(step_s, 7), "unit": "s", "ms_per_step": round(ms_per_step, 4),
                "alg_bytes_per_step": alg_bytes, "hbm_frac": round(alg_bytes / step_s / 1e9 / hbm_peak, 4),
                "clocks": clk.summary(), "timing": "CUDA events around CUDA-graph replays of the whole step",
                "alu_roof": alu_roof(ctx, st, stage_ms, clk.summary()),
                "stage_ms_eager": {k: round(v, 4) for k, v in zip(("fwd", "mac", "tail"), stage_ms)}}

    # ---- per-stage live timing (eager stage calls, launches pre-queued behind a sleep) ----
    stage_ms = stage_profile(ctx, st, K, dev)

    # ---- e2e: host buffers, H2D + public API + D2H every step ----
    e2e = None if args.no_e2e else run_e2e(ctx, st, K, dev, share_buf, world, runner, drawn=drawn)

    # ---- f4: online NTT preprocessing (weights in coefficient form, transformed in each call) ----
    online = None if args.no_online else run_online(ctx, st, K, args.warmup, dev, world, runner)

    # ---- f2: extracted outputs (modulus switch + designated coefficients) ----
    lwe = run_lwe(ctx, st, K, args.warmup, dev, world, runner, drawn=drawn, priority=hi)
    if not args.no_e2e:  # the same step end to end, sending back only the extracted outputs
        lwe["e2e"] = run_e2e(ctx, st, K, dev, share_buf, world, runner, lwe_keep=ctx.L // 2, drawn=drawn)

    # ---- f3: the ResNet-50 fully-connected layer through secn_he_fc ----
    fc_leg = run_fc(ctx, K, args.warmup, dev, world)

    if rank != 0:
        return None

    # ---- derived numbers ----
    n_ntt = sum((d["plan"].G * d["plan"].S * world + d["plan"].M * d["plan"].S) * 2 * L for d in st)  # limb NTTs per step
    # NTT, (mask draw,) MAC(+INTT 0-7), INTT tail(+mask, share)
    launches_per_step = sum(4 if drawn else 3 for d in st if d["mc"] > 0)
    sb = {s: sum(stage_bytes(d["pl"], L, n, wbytes)[s] for d in st if d["mc"] > 0) for s in range(3)}
    names = {0: "k_ntt_fwd (A6 share add + A1 NTT)", 1: "k_mac (A4 NTT-domain MAC + INTT levels 0-7)",
             2: "k_ntt_inv_tail (A2 INTT levels 8-11 + A7 mask)"}
    dom = max(range(3), key=lambda s: stage_ms[s])
    n_layers_active = sum(1 for d in st if d["mc"] > 0)
    achieved = sb[dom] / (stage_ms[dom] / 1e3) / 1e9
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture (per launch,
    # its largest launch: conv10), next to that launch's algorithmic bytes
    tr = None
    trf = ROOT / "profiles" / "kmac_traffic.json"
    if dom == 1 and trf.exists():
        tr = json.loads(trf.read_text())
    roofline = {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                "traffic": tr["dram_bytes_per_launch"] if tr else None,
                "traffic_note": (f"ncu DRAM read+write of one {tr['layer']} launch ({tr.get('dram_GBps_ncu')} GB/s in "
                                 f"{tr['duration_us_ncu']} us); algorithmic bytes of that launch "
                                 f"{tr['algorithmic_bytes_per_launch']}; integer-multiply (fmaheavy) pipe "
                                 f"{tr['fmaheavy_pct_of_peak_elapsed']}% busy ({tr['source']})") if tr else None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "bytes_per_step": sb[dom], "launches_per_step": n_layers_active,
                "avg_launch_us": round(stage_ms[dom] / n_layers_active * 1e3, 2),
                "stage_ms": {names[s]: round(stage_ms[s], 4) for s in range(3)},
                "stage_GBps": {names[s]: round(sb[s] / (stage_ms[s] / 1e3) / 1e9, 1) for s in range(3)}}
    roofline["alu_roof"] = alu_roof(ctx, st, stage_ms, clk.summary())
    # the whole step against its byte floors, and every kernel's pipes and stalls, from the committed
    # ncu capture of one step (tools/gpu_step_ncu.sh -> profiles/*_step_ncu.json)
    bytemin = sum(algorithmic_bytes(ctx.plan(d["lay"].C, d["lay"].H, d["lay"].W, d["lay"].M, d["lay"].k,
                                             stride=d["lay"].stride, pad=d["lay"].pad, rule=0), L, n, wbytes, drawn)
                  for d in st)
    roofline["step"] = {"alg_bytes_executed_plans": alg_bytes, "alg_bytes_byte_min_plans": bytemin,
                        "hbm_frac_executed_plans": round(alg_bytes / step_s / 1e9 / (hbm_peak * world), 4),
                        "hbm_frac_byte_min_plans": round(bytemin / step_s / 1e9 / (hbm_peak * world), 4)}
    snc = sorted((ROOT / "profiles").glob("*_step_ncu.json"))
    if snc and world == 1:
        sj = json.loads(snc[-1].read_text())
        roofline["step"].update({
            "dram_traffic_ncu": sj["step_dram_bytes"],
            "traffic_over_alg_bytes": round(sj["step_dram_bytes"] / alg_bytes, 3),
            "ncu_source": f"profiles/{snc[-1].name} (one eager step, kernels serialised by ncu)",
            "kernels": {k: {f: v for f, v in kv.items() if f in ("issue_active_pct", "pipe_alu_pct", "pipe_fma_pct",
                                                                 "warps_active_pct", "dram_bytes", "top_stalls_per_issue")}
                        for k, kv in sj["kernels"].items()}})
    out = {
        "metric": net_info(args.net)[0], "value": round(step_s, 7), "unit": "s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": f"u{ctx.word_bits}", "data": "synthetic (seeded uniform cts/shares/masks, "
        "He-normal 37-bit/scale-12 kernels)",
        "config": {"workload": net_info(args.net)[1],
                   "N": n, "limbs": L, "primes": [hex(q) for q in ctx.primes], "t_bits": t_bits,
                   "parallelism": (f"(output channel x spatial block) rectangles over {world} ranks "
                                   "(paper_2506_11586_b200/dist.partition)" if world > 1 else "1 GPU"),
                   "mask": ({"inline": "drawn + encoded on the device inside every layer call (secn32_he_conv2d_gen, "
                                       "Philox4x32-10, reading R17)",
                             "lookahead": "drawn + encoded on the device (secn_mask_encode, Philox4x32-10, reading R17) "
                                          "on a side stream one layer ahead of the chain, added by secn32_he_conv2d_em",
                             "ahead": "drawn + encoded on the device (secn_mask_encode, Philox4x32-10, reading R17) for "
                                      "every layer at the start of the step on a side stream, added by "
                                      "secn32_he_conv2d_em"}[msched]
                            if drawn else "caller input r (secn32_he_conv2d_ex)"), "l2": (f"inputs {alg_bytes / 1e9:.2f} GB/step >> 126 MB L2 (no flush)" if alg_bytes > 5e8 else
                          "step footprint below 4x L2: timing includes L2 reuse across replays"),
                   "timing": "CUDA events around CUDA-graph replays of the whole step",
                   "layer_overlap": {"none": "none: every layer in network order on one stream",
                                     "staged": "staged: layers reading the same input tensor (fire e1/e3, ResNet "
                                               "c1/ds) run each launch group side by side, joined between groups",
                                     "free": "free: layers reading the same input tensor (fire e1/e3, ResNet "
                                             "c1/ds) on two streams; the rest in network order"}[args.overlap]},
        "throughput": {"ntt_per_s": round(n_ntt / step_s, 1), "alg_bytes_per_step": alg_bytes,
                       "alg_GBps": round(alg_bytes / step_s / 1e9, 1),
                       "hbm_frac": round(alg_bytes / step_s / 1e9 / (hbm_peak * world), 4),
                       "offline_preprocess_s": round(offline_s, 5), "wall_s_timed_region": round(wall, 4)},
        "roofline": roofline,
        "per_layer_stage_us": stage_profile.per_layer_us,
        "gpu_launches": launches_per_step * K,
        "clocks": clk.summary(),
        "e2e": e2e, "online_ntt_preprocessing": online, "extracted_outputs": lwe, "fc": fc_leg,
        "context": {"paper_gpu_online_s": 2.26, "paper_gpu_hw": "RTX A6000 + Troy (PAPER.md:476)",
                    "paper_cpu_online_s": 3.09},
    }
    if not args.no_cpu_baseline and world == 1:
        frac = args.cpu_frac if args.cpu_frac is not None else default_cpu_frac(args.net)
        out["cpu_baseline"] = cpu_baseline(st, ctx, frac, dev, wbytes, args.seed, drawn)
    return out


# Calibrated integer throughputs (ops per clock per SM; profiles/r01_calib_intpipe.txt, tools/calib):
# a lazy modular butterfly and a 64x64 -> 128-bit multiply-accumulate for 64-bit words, an exact
# 32-bit Shoup product for 32-bit words (one butterfly), IMAD.WIDE for a 32-bit MAC.
CALIB = {64: {"bfly": 2.97, "mac": 3.69}, 32: {"bfly": 15.86, "mac": 27.95}}


def alu_roof(ctx, st, stage_ms, clocks):
    """Each stage's integer-ALU floor -- its modular butterflies and multiply-accumulates at the
    calibrated rates on every SM at the sampled SM clock -- against its eager device time."""
    L, n = ctx.L, ctx.n
    logn = n.bit_length() - 1
    rate = CALIB[ctx.word_bits]
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    hz = (clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0) * 1e6
    bf = n // 2
    fwd_b = sum(2 * d["pl"].G * d["pl"].S * L * bf * logn for d in st if d["mc"] > 0)
    out_polys = sum(2 * d["pl"].M * d["pl"].S * L for d in st if d["mc"] > 0)
    macs = sum(2 * d["pl"].M * d["pl"].G * d["pl"].S * L * n for d in st if d["mc"] > 0)
    floor_ms = [fwd_b / (rate["bfly"] * sms * hz) * 1e3,
                (macs / rate["mac"] + out_polys * bf * 8 / rate["bfly"]) / (sms * hz) * 1e3,
                out_polys * bf * (logn - 8) / (rate["bfly"] * sms * hz) * 1e3]
    return {"rates_per_clk_per_sm": rate, "source": "profiles/r01_calib_intpipe.txt (tools/calib/intbench.cu)",
            "sm_clock_mhz": hz / 1e6, "sms": sms,
            "stages": {k: {"floor_ms": round(f, 4), "measured_ms": round(m, 4), "frac": round(f / m, 3) if m else None}
                       for k, f, m in zip(("fwd (A6 + A1 NTT)", "mac (A4 MAC + INTT levels 0-7)",
                                           "tail (INTT levels 8.. + mask)"), floor_ms, stage_ms)},
            "step_floor_ms": round(sum(floor_ms), 4)}


def stage_profile(ctx, st, K, dev):
    """Per-launch-group device time, CUDA events on the launching stream around each stage;
    the whole step's launches are enqueued behind a spin kernel so no host gap is timed."""
    stream = torch.cuda.current_stream(dev)

    def run(evs):
        for li, d in enumerate(st):
            if d["mc"] <= 0:
                continue
            a = (d["pl"], d["ct"], d["w"], d["x0"], d["r"], d["out"], d["ws"])
            evs[li][0].record(stream)
            ctx.he_conv2d_stage(0, a[0], a[1], a[2], a[3], a[4], a[5], a[6])
            evs[li][1].record(stream)
            ctx.he_conv2d_stage(1, a[0], a[1], a[2], a[3], a[4], a[5], a[6])
            evs[li][2].record(stream)
            ctx.he_conv2d_stage(2, a[0], a[1], a[2], a[3], a[4], a[5], a[6])
            evs[li][3].record(stream)
            ctx.extract_share(d["pl"], d["r"], out=d["y0"])

    mk = lambda: [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in st]  # noqa: E731
    torch.cuda.synchronize()
    t = time.perf_counter()
    run(mk())
    host_s = time.perf_counter() - t
    torch.cuda.synchronize()
    tot = [0.0, 0.0, 0.0]
    per_layer = {d["lay"].name: [0.0, 0.0, 0.0] for d in st}
    for _ in range(K):
        evs = mk()
        torch.cuda._sleep(int(2.5e9 * (2 * host_s + 1e-3)))
        run(evs)
        torch.cuda.synchronize()
        for li, d in enumerate(st):
            if d["mc"] > 0:
                for s in range(3):
                    dt = evs[li][s].elapsed_time(evs[li][s + 1])
                    tot[s] += dt
                    per_layer[d["lay"].name][s] += dt
    stage_profile.per_layer_us = {k: [round(v * 1e3 / K, 1) for v in vs] for k, vs in per_layer.items()}
    return [x / K for x in tot]


def ctx_lib():
    from paper_2506_11586_b200 import secn

    return secn.lib()


def graph_ms(fn, K, warmup, dev, world, priority=0):
    """Captures fn() in a CUDA graph and returns the device ms per replay (max over ranks)."""
    for _ in range(max(warmup, 3)):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev, priority=priority)
    cap.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.graph(g, stream=cap):
        fn()
    torch.cuda.synchronize()
    for _ in range(max(warmup, 3)):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a.record()
    for _ in range(K):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / K], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    del g
    return float(ms.item())


def _leg_overlap(runner):
    """The schedule a secondary leg ran under: GroupRunner overlaps its groups on two streams; the
    StagedGroupRunner has no staged form of these entry points and runs them in network order."""
    from paper_2506_11586_b200.schedule import StagedGroupRunner
    if isinstance(runner, StagedGroupRunner) or all(len(g) == 1 for g in runner.groups):
        return "none: network order"
    return "free: layers reading the same input on two streams"


def run_online(ctx, st, K, warmup, dev, world, runner):
    """SURVEY.md §8f row 4 / PAPER.md:433, :498: the same step with the weights held in coefficient
    form (the tiny quantised kernels) and packed + transformed inside every secn32_he_conv2d_online
    call, instead of the offline-preprocessed NTT-domain weights."""
    for d in st:
        if d["mc"] > 0:
            d["ws_on"] = torch.empty((ctx.online_workspace_bytes(d["pl"]) + 7) // 8, dtype=torch.int64, device=dev)

    def layer_online(i):
        d = st[i]
        if d["mc"] > 0:
            ctx.he_conv2d_online(d["pl"], d["ct"], d["K"], x0=d["x0"], r=d["r"], out=d["out"], workspace=d["ws_on"],
                                 y0=d["y0"])

    ms = graph_ms(lambda: runner(layer_online), K, warmup, dev, world)
    for d in st:
        d.pop("ws_on", None)
    torch.cuda.empty_cache()
    held = sum(d["K"].numel() * 8 for d in st if d["mc"] > 0)
    return {"value": round(ms / 1e3, 7), "unit": "s", "ms_per_step": round(ms, 4),
            "weights_held_bytes": held, "weights_held_offline_bytes": sum(d["w"].numel() * d["w"].element_size()
                                                                            for d in st if d["mc"] > 0),
            "path": "secn_he_conv2d_online: pack + NTT of the weights, then share add + NTT, MAC, INTT + mask",
            "layer_overlap": _leg_overlap(runner)}


def run_lwe(ctx, st, K, warmup, dev, world, runner, drawn=False, priority=0):
    """the same step returning extracted outputs (secn32_he_conv2d_lwe: the
    INTT tail switches every output ct to half of its limbs and keeps the b component only at the
    designated coefficients), i.e. what Cheetah's server sends back. With the drawn mask, the same
    schedule as the main step: every layer's mask encoded at the start on a side stream, each layer
    through secn32_he_conv2d_lwe_em after its mask's event."""
    keep = ctx.L // 2
    for d in st:
        if d["mc"] > 0:
            pl = d["pl"]
            d["ws_lwe"] = torch.empty((int(ctx_lib().secn_he_conv2d_lwe_workspace(ctx._h, ctypes.byref(pl))) + 7) // 8,
                                      dtype=torch.int64, device=dev)
            d["lwe_out"] = (ctx.empty(d["mc"] * pl.S, keep, ctx.n), ctx.empty(d["mc"], pl.OH, pl.OW, keep))
    mstream = torch.cuda.Stream(dev)
    mev = [torch.cuda.Event() for _ in st]

    def layer_lwe(i):
        d = st[i]
        if d["mc"] > 0 and drawn:
            torch.cuda.current_stream().wait_event(mev[i])
            ctx.he_conv2d_lwe_em(d["pl"], d["ct"], d["w"], keep, d["em"], x0=d["x0"], workspace=d["ws_lwe"],
                                 out=d["lwe_out"])
        elif d["mc"] > 0:
            ctx.he_conv2d_lwe(d["pl"], d["ct"], d["w"], keep, x0=d["x0"], r=d["r"], y0=d["y0"],
                              workspace=d["ws_lwe"], out=d["lwe_out"])

    def step():
        if drawn:
            mstream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(mstream):
                for i, d in enumerate(st):
                    if d["mc"] > 0:
                        ctx.mask_encode(d["pl"], gen=d["gen"], out=d["em"], y0=d["y0"])
                        mev[i].record(mstream)
        runner(layer_lwe)
        if drawn:
            torch.cuda.current_stream().wait_stream(mstream)

    ms = graph_ms(step, K, warmup, dev, world, priority=priority)
    out_bytes = sum(a.numel() * a.element_size() + b.numel() * b.element_size()
                    for a, b in (d["lwe_out"] for d in st if d["mc"] > 0))
    full_bytes = sum(d["out"].numel() * d["out"].element_size() for d in st if d["mc"] > 0)
    for d in st:
        d.pop("ws_lwe", None)
        d.pop("lwe_out", None)
    torch.cuda.empty_cache()
    return {"value": round(ms / 1e3, 7), "unit": "s", "ms_per_step": round(ms, 4), "keep_limbs": keep,
            "output_bytes_per_step": out_bytes, "full_ct_output_bytes_per_step": full_bytes,
            "path": ("secn_mask_encode ahead (drawn mask) + secn32_he_conv2d_lwe_em: share add + NTT, MAC, INTT tail + "
                     "mask + modulus switch + extraction" if drawn else
                     "secn32_he_conv2d_lwe: share add + NTT, MAC, INTT tail + mask + modulus switch + extraction"),
            "layer_overlap": _leg_overlap(runner)}


def run_fc(ctx, K, warmup, dev, world, n_i=2048, n_o=1000, seed=11):
    """ResNet-50's fully-connected layer (2048 -> 1000) through secn_he_fc
    (share add + NTT, MAC, INTT + mask + server share), weights preprocessed offline."""
    p = ctx.fc_plan(n_i, n_o)
    g = inputs.rng(seed)
    L, n = ctx.L, ctx.n
    ct = inputs.uniform_residues(g, (p.G, 2), ctx.primes, n)
    ctd = torch.from_numpy(ct.view(np.int64) if ctx.word_bits == 64 else ct.astype(np.uint32).view(np.int32)).to(dev)
    x0 = torch.from_numpy(inputs.uniform_below(g, (p.G, n), 1 << ctx.t_bits).view(np.int64)).to(dev)
    Wm = inputs.quantized_kernel(g, n_o, n_i, 1, 1).reshape(n_o, n_i)
    w = ctx.fc_preprocess_weights(p, torch.from_numpy(Wm.view(np.int64)).to(dev))
    r = torch.from_numpy(inputs.uniform_below(g, (p.M, n), 1 << ctx.t_bits).view(np.int64)).to(dev)
    out = ctx.empty(p.M, 2, L, n)
    y0 = torch.empty(n_o, dtype=torch.int64, device=dev)
    ms = graph_ms(lambda: ctx.he_fc(p, ctd, w, x0=x0, r=r, out=out, y0=y0), K, warmup, dev, world)
    wb = ctx.word_bits // 8
    alg = wb * L * n * (2 * p.G + p.M * p.G + 2 * p.M) + 8 * n * p.M + 8 * n * p.G
    return {"layer": f"resnet50 fc {n_i}->{n_o}", "plan": {"nib": p.nib, "nob": p.nob, "G": p.G, "M": p.M},
            "value": round(ms / 1e3, 8), "unit": "s", "alg_bytes": alg,
            "hbm_frac": round(alg / (ms / 1e3) / 1e9 / peaks()[0], 4), "launches": 3}


def run_e2e(ctx, st, K, dev, share_buf, world, runner, lwe_keep=None, drawn=False):
    """Same metric end to end through the public API: every step copies that step's inputs
    (ct_in, x0, r) host->device from pinned memory, runs secn_he_conv2d_ex (ciphertexts and the
    server's shares) per layer, and copies the output ciphertexts and shares device->host.
    With lwe_keep, the call is secn32_he_conv2d_lwe instead and the device->host copy is the
    extracted, modulus-switched outputs (what Cheetah's server sends)."""
    host = []
    h2d = d2h = 0
    for d in st:
        if d["mc"] <= 0:
            continue
        if lwe_keep:
            pl = d["plan"]
            wsf = ctx_lib().secn_he_conv2d_lwe_gen_workspace if drawn else ctx_lib().secn_he_conv2d_lwe_workspace
            d["ws_lwe"] = torch.empty((int(wsf(ctx._h, ctypes.byref(d["pl"]))) + 7) // 8, dtype=torch.int64, device=dev)
            d["lwe_out"] = (ctx.empty(d["mc"] * pl.S, lwe_keep, ctx.n), ctx.empty(d["mc"], pl.OH, pl.OW, lwe_keep))
        ct = np.ascontiguousarray(d["ct_h"])
        ct = ct.view(np.int64) if d["ct"].dtype == torch.int64 else ct.astype(np.uint32).view(np.int32)
        h = {"ct": torch.from_numpy(ct).pin_memory(),
             "x0": torch.from_numpy(np.ascontiguousarray(d["x0_h"]).view(np.int64)).pin_memory()}
        S = d["plan"].S
        if not drawn:  # a caller-supplied mask is an input that crosses PCIe every step
            h["r"] = torch.from_numpy(np.ascontiguousarray(d["r_h"][d["m0"] * S:(d["m0"] + d["mc"]) * S]).view(np.int64)).pin_memory()
        if lwe_keep:
            h["lwe_out"] = tuple(torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in d["lwe_out"])
            h["out"] = torch.empty(0, dtype=d["out"].dtype)
            d2h += sum(t.numel() * t.element_size() for t in h["lwe_out"])
        else:
            h["out"] = torch.empty(d["out"].shape, dtype=d["out"].dtype).pin_memory()
            d2h += h["out"].numel() * h["out"].element_size()
        h["y0"] = torch.empty(d["y0"].shape, dtype=torch.int64).pin_memory()
        h2d += sum(h[k].numel() * h[k].element_size() for k in ("ct", "x0", "r") if k in h)
        d2h += h["y0"].numel() * 8
        host.append((d, h))

    # Three streams, as a serving loop would run them: host->device copies, the library calls and
    # device->host copies. Layer i's copies overlap other layers' compute and each other (the two
    # PCIe directions are independent). Per layer, the next step's input copy waits until this
    # step's call has read the inputs, and the next call waits until this step's outputs are out.
    cs = torch.cuda.current_stream(dev)
    hs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    comp_done = {}
    out_done = {}

    def step():
        for d, h in host:
            k = id(d)
            if k in comp_done:
                hs.wait_event(comp_done[k])
            with torch.cuda.stream(hs):
                d["ct"].copy_(h["ct"], non_blocking=True)
                d["x0"].copy_(h["x0"], non_blocking=True)
                if not drawn:
                    d["r"].copy_(h["r"], non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(hs)
            cs.wait_event(e_in)
            if k in out_done:
                cs.wait_event(out_done[k])
            if lwe_keep and drawn:
                ctx.he_conv2d_lwe_gen(d["pl"], d["ct"], d["w"], lwe_keep, d["gen"], x0=d["x0"], y0=d["y0"],
                                      workspace=d["ws_lwe"], out=d["lwe_out"])
            elif lwe_keep:
                ctx.he_conv2d_lwe(d["pl"], d["ct"], d["w"], lwe_keep, x0=d["x0"], r=d["r"], y0=d["y0"],
                                  workspace=d["ws_lwe"], out=d["lwe_out"])
            elif drawn:
                ctx.he_conv2d_gen(d["pl"], d["ct"], d["w"], d["gen"], x0=d["x0"], out=d["out"], workspace=d["ws_gen"],
                                  y0=d["y0"])
            else:
                ctx.he_conv2d(d["pl"], d["ct"], d["w"], x0=d["x0"], r=d["r"], out=d["out"], workspace=d["ws"],
                              y0=d["y0"])
            comp_done[k] = torch.cuda.Event()
            comp_done[k].record(cs)
            ds.wait_event(comp_done[k])
            with torch.cuda.stream(ds):
                if lwe_keep:
                    for hd, dd in zip(h["lwe_out"], d["lwe_out"]):
                        hd.copy_(dd, non_blocking=True)
                else:
                    h["out"].copy_(d["out"], non_blocking=True)
                h["y0"].copy_(d["y0"], non_blocking=True)
                out_done[k] = torch.cuda.Event()
                out_done[k].record(ds)

    def drain():  # the compute stream waits for every copy issued so far
        cs.wait_stream(hs)
        cs.wait_stream(ds)

    for _ in range(2):
        step()
    drain()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    a.record(cs)
    hs.wait_event(a)
    ds.wait_event(a)
    for _ in range(K):
        step()
    drain()
    b.record(cs)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / K], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # the host copies of the last step equal the device results (every step has the same inputs)
    outs = (lambda d, h: zip(h["lwe_out"], d["lwe_out"])) if lwe_keep else (lambda d, h: [(h["out"], d["out"])])
    same = all(all(torch.equal(ho, do.cpu()) for ho, do in outs(d, h)) and torch.equal(h["y0"], d["y0"].cpu())
               for d, h in host)
    for d, _ in host:
        d.pop("ws_lwe", None)
        d.pop("lwe_out", None)
    call = (f"secn32_he_conv2d_lwe{'_gen' if drawn else ''} (keep {lwe_keep} limbs)" if lwe_keep else
            ("secn32_he_conv2d_gen" if drawn else "secn32_he_conv2d_ex"))
    return {"value": round(float(ms.item()) / 1e3, 6), "unit": "s", "host_copies_match_device": same,
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "path": f"pinned host -> {call} -> pinned host; H2D, calls and D2H on three streams (per-layer "
                    "events), so copies of one layer overlap the other layers' compute and each other"
                    + ("; the mask is drawn on the device (no r crosses PCIe)" if drawn else "")}


# ------------------------------------------------------------------------------------------
# the oracle on the host cores (cpu_baseline and the --impl reference arm). Neither leg imports
# the product package: the oracle plans every layer itself (reading R6b, oracle/packing.py) --
# the GPU arm asserts that its library chose the same window -- and packs the weights once per
# layer (the offline setup, untimed, as the GPU arm's weight preprocessing is); the timed part is
# the online server computation over every output ciphertext of the network.

def oracle_states(net, P, words64, seed, drawn=True):
    """Per layer: the oracle's plan, the seeded inputs (identical to the GPU arm's) and the
    sparse plaintext polys. With drawn, r is left to oracle_run, which draws it from the oracle's
    Philox4x32-10 (oracle/philox.py) inside the timed region, as the GPU arm draws it in its step."""
    from oracle import packing

    states = []
    for li, lay in enumerate(net):
        opl = packing.plan_conv(lay.C, lay.H, lay.W, lay.M, lay.k, lay.k, lay.stride, lay.pad, P.n, words64,
                                rule="time")
        ct, x0, K, r = layer_inputs(P.primes, P.n, P.t_bits, lay, opl.G, opl.S, opl.M, seed * 1000 + li)
        kp = packing.sparse(packing.kernel_polys(K, opl, P.n))
        states.append({"lay": lay, "opl": opl, "ct_h": ct, "x0_h": x0, "K_h": K, "r_h": None if drawn else r,
                       "kp": kp, "gen": (mask_seed(seed), li) if drawn else None})
    return states


def oracle_chunks(states, parts, frac=1.0):
    """Splits the network's output ciphertexts -- flattened in (layer, ct) order, the first
    ceil(frac * n_out) of every layer -- into `parts` consecutive chunks. Returns per chunk a list
    of (layer index, lo, hi) ranges."""
    flat = []
    for li, d in enumerate(states):
        n_out = d["opl"].M * d["opl"].S
        flat.append((li, n_out if frac >= 1 else max(1, math.ceil(frac * n_out))))
    total = sum(k for _, k in flat)
    bounds = [total * i // parts for i in range(parts + 1)]
    chunks, pos = [], 0
    cum = []
    for li, k in flat:
        cum.append((li, pos, pos + k))
        pos += k
    for i in range(parts):
        lo, hi = bounds[i], bounds[i + 1]
        rs = [(li, max(lo, a) - a, min(hi, b) - a) for li, a, b in cum if max(lo, a) < min(hi, b)]
        chunks.append(rs)
    return chunks, total


def oracle_run(states, P, ranges, check=None):
    """Runs the oracle's server computation on the given (layer, lo, hi) output ranges.
    Returns (measured seconds, outputs, parity mismatches); `check(li, lo, hi)` returns the GPU's
    outputs [hi-lo][2][L][N] as uint64 (or None) to compare word for word (not timed)."""
    from oracle import he, philox

    dt, n, bad = 0.0, 0, 0
    for li, lo, hi in ranges:
        d = states[li]
        o = d["opl"]
        sel = np.zeros(o.M * o.S, np.uint8)
        sel[lo:hi] = 1
        t0 = time.perf_counter()
        r = d["r_h"]
        if d["gen"] is not None:  # the mask rows of these outputs, drawn as the GPU draws them
            r = np.zeros((o.M * o.S, P.n), np.uint64)
            r[lo:hi] = philox.mask(d["gen"][0], d["gen"][1], hi - lo, P.n, P.t_bits, ct0=lo)
        ref = he.server_mac_sparse(d["ct_h"], d["x0_h"], d["kp"], r, o.G, o.S, o.M, P, sel=sel)
        dt += time.perf_counter() - t0
        n += hi - lo
        if check is not None:
            got = check(li, lo, hi)
            if got is not None:
                bad += int((got != ref[lo:hi]).sum())
        del ref
    return dt, n, bad


def default_cpu_frac(net):
    """The oracle covers every output ciphertext of SqueezeNet (~1 min on 16 cores); ResNet-50
    (1e12 modular products) runs on the first 2% of each layer's outputs, labelled extrapolated."""
    return 0.02 if net == "resnet50" else 1.0


def cpu_baseline(st, ctx, frac, dev, wbytes, seed, drawn=True):
    """The oracle on this box's host cores over the whole network (frac = 1: every output
    ciphertext, measured, no extrapolation), on the GPU arm's seeded inputs; every output word is
    also compared with the GPU's (parity_mismatched_words)."""
    from oracle import _c
    from oracle.params import Params

    P = Params(primes=ctx.primes)
    states = oracle_states([d["lay"] for d in st], P, ctx.coef_words64, seed, drawn)
    for d, o in zip(st, states):  # the oracle planned every layer itself: the library must agree
        assert (o["opl"].Hw, o["opl"].Ww, o["opl"].decim == 2, o["opl"].G, o["opl"].S) == \
            (d["plan"].Hw, d["plan"].Ww, d["plan"].decim == 2, d["plan"].G, d["plan"].S), d["lay"].name

    def check(li, lo, hi):
        d = st[li]
        if d["mc"] != d["plan"].M:
            return None
        torch.cuda.synchronize()
        x = d["out"][lo:hi].cpu().numpy()
        return x.view(np.uint64) if wbytes == 8 else x.view(np.uint32).astype(np.uint64)

    (ranges,), total = oracle_chunks(states, 1, frac)
    dt, n, bad = oracle_run(states, P, ranges, check)
    n_all = sum(o["opl"].M * o["opl"].S for o in states)
    full = n == n_all
    return {"value": round(dt if full else dt * n_all / n, 3), "unit": "s", "cores": _c.lib().orc_num_threads(),
            "kind": "oracle",
            "sample": (f"the whole network: all {n} output ciphertexts of {len(states)} layers, one measured pass "
                       f"({dt:.2f} s; weights packed once per layer beforehand, untimed)" if full else
                       f"the first {frac:.1%} of every layer's outputs ({n} of {n_all} ciphertexts) measured in "
                       f"{dt:.2f} s, extrapolated by output count"),
            "parity_mismatched_words": bad, "parity_words_compared": n * 2 * ctx.L * ctx.n}


def run_reference(args, world, rank):
    """--impl reference: the oracle (plain C schoolbook, OpenMP) on the host cores, same metric.
    The K timed steps split the network's output ciphertexts into K consecutive chunks, so they
    cover the whole network exactly once: `value` is the measured time of one full pass (the sum
    of the K steps), not an extrapolation. Imports nothing from the product package."""
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    from oracle import _c
    from oracle import params as oparams
    from oracle.params import Params

    net = layers.network(args.net)
    P = Params(primes=oparams.DEFAULT_PRIMES if args.word_bits == 64 else oparams.PRIMES32)
    words64 = max(1, P.L * args.word_bits // 64)
    states = oracle_states(net, P, words64, args.seed, args.mask == "device")
    frac = args.cpu_frac if args.cpu_frac is not None else default_cpu_frac(args.net)
    small = min(range(len(states)), key=lambda i: states[i]["opl"].M * states[i]["opl"].S)
    for _ in range(args.warmup):  # one output ciphertext of the smallest layer
        oracle_run(states, P, [(small, 0, 1)])
    chunks, total = oracle_chunks(states, max(1, args.steps), frac)
    times, n_done = [], 0
    for rs in chunks:
        dt, n, _ = oracle_run(states, P, rs)
        times.append(dt)
        n_done += n
    n_all = sum(o["opl"].M * o["opl"].S for o in states)
    meas = sum(times)
    v = meas if n_done == n_all else meas * n_all / n_done
    thr = _c.lib().orc_num_threads()
    sample = (f"the whole network once: {n_all} output ciphertexts of {len(states)} layers split into {len(chunks)} "
              f"consecutive chunks, one per timed step; value = measured sum ({meas:.2f} s)" if n_done == n_all else
              f"the first {frac:.1%} of every layer's outputs ({n_done} of {n_all}), measured {meas:.2f} s, "
              f"extrapolated by output count")
    out = {"impl": "reference", "metric": net_info(args.net)[0], "value": round(v, 3), "unit": "s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(meas / max(1, len(chunks)) * 1e3, 1),
           "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": f"u{args.word_bits}",
           "data": "synthetic",
           "config": {"workload": net_info(args.net)[1], "N": P.n, "limbs": P.L, "t_bits": P.t_bits},
           "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": thr, "kind": "oracle", "sample": sample},
           "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
