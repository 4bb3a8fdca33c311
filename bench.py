#!/usr/bin/env python
"""bench.py — the MASQuant hot path on B200, one JSON line on rank 0.

Step = one pass of every SURVEY §8(a) row over one calibration batch of the c3 workload
(BASELINE.json configs[2], the Qwen2.5-VL-7B shapes the north-star's 60%-of-INT8-peak target is
quoted on): for each of the layer's four (fused) linears
    A1 masq_calibrate_stats -> [NCCL MAX/SUM all-reduce of R / counts, batched, N>1]
    A2 masq_init_factors -> masq_calib_layer, one fused call per linear:
       A3 Q(S_m W) for every modality from one read of W (set 0 = the forward's Q(S_t W)),
       A4-A7 forward (W4A8, CMC rank r for image tokens), A8 X W and the loss (the forward's
       activation codes gathered into modality-grouped order)
       -> [NCCL SUM all-reduce of the loss sums / counts, batched, N>1] -> masq_loss_finalize
Weak scaling: every rank calibrates its own 16384-token batch (token-sharded data parallel).

A separate "n1" block times SURVEY §8(f)'s first next row on the same inputs, outside the
step: one S-optimisation iteration per linear = masq_calib_loss_grad (loss + straight-through
gradient, global-count normalised) -> [NCCL SUM of the gradient, N>1] -> masq_adam_step.

value = tokens of all ranks / device time of K steps (CUDA events, max over ranks).
--impl reference times the CPU oracle (oracle/) on a bounded sample instead.
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "calibration tokens/sec and quantized-linear TOPS (% of B200 INT8 peak), 1/2/4/8 GPU"
CFG = "c3"
CI = 2                      # configs[2]
WBITS, ABITS = 4, 8
N_MOD = 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="masq", choices=["masq", "reference"])
    ap.add_argument("--rank-cmc", type=int, default=None, help="CMC rank r (0 disables; default c3 64, c2 0)")
    ap.add_argument("--tokens", type=int, default=None, help="tokens per GPU (default c3 16384, c2 4096)")
    ap.add_argument("--linears", default="qkv,o,gate_up,down")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-n1", action="store_true", help="skip the N1 S-optimisation step timing")
    ap.add_argument("--streams", type=int, default=1,
                    help="CUDA streams the timed step's linears are spread over (default 1: every kernel's CUDA-event "
                         "duration is its own, which the per-kernel table and roofline need; the line also carries an "
                         "'overlapped' block timing the same step on 2 streams, where one linear's HBM-bound kernels "
                         "run beside another's GEMM; c4/c4s use 2)")
    ap.add_argument("--nvtx", action="store_true",
                    help="NVTX ranges around the step's phases (stats / per-linear calib_layer), for ncu --nvtx filters")
    ap.add_argument("--graph", action="store_true",
                    help="replay the step as one captured CUDA graph (N=1; measured slower here: the launch "
                         "gaps are ~2%% of the step and the captured profiler event nodes cost more)")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no baselines)")
    ap.add_argument("--c5-n", type=int, default=18944, help="c5: output channels of the d=3584 linear")
    ap.add_argument("--workload", default="c3", choices=["c2", "c3", "c4", "c4s", "c5"],
                    help="c3: one Qwen2.5-VL-7B layer, every §8(a) row (default); c2: the same step on one "
                         "Qwen2.5-Omni-3B layer (text/image/audio, W8A8, 4096 tokens, r = 0); c4 (= c4s): 28-layer "
                         "calibration sweep with 2 real S-optimisation epochs per layer (N1: loss + "
                         "straight-through gradient + Adam)")
    ap.add_argument("--layers", type=int, default=28, help="c4: number of decoder layers")
    args = ap.parse_args()
    configure(args)
    return args


def configure(args):
    """Select the layer workload: c3 (BASELINE configs[2], default) or c2 (configs[1])."""
    global CFG, CI, WBITS, ABITS, N_MOD
    if args.workload == "c2":
        CFG, CI, WBITS, ABITS, N_MOD = "c2", 1, 8, 8, 3
    cfg = synth.CONFIGS[CFG]
    if args.tokens is None:
        args.tokens = 16384 if args.workload in ("c3", "c4", "c4s", "c5") else cfg["T"]
    if args.rank_cmc is None:
        args.rank_cmc = 64 if args.workload != "c2" else cfg["r"]


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return dict(hbm=float(j["hbm_gbs"]), bf16=float(j["bf16_tflops"]),
                    bf16_sus=float(j.get("bf16_tflops_sustained", j["bf16_tflops"])), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


# --------------------------------------------------------------------------- inputs
def layer_linears(names):
    table = {k: (d, n) for k, d, n in synth.LAYER_LINEARS[CFG]}
    return [(k, *table[k]) for k in names]


def make_host_inputs(T, rank, linears, r):
    cfg = synth.CONFIGS[CFG]
    ids = synth.modality_ids(cfg["pattern"], T=T)
    out = []
    for li, (name, d, n) in enumerate(linears):
        X = synth.activations(ids, d, N_MOD, synth.seed_for(CI, li, 0) + 100000 * rank)
        W = synth.weight(d, n, synth.seed_for(CI, li, 1))
        L1, L2 = synth.lowrank(d, n, r, N_MOD, synth.seed_for(CI, li, 2)) if r > 0 else (None, None)
        out.append(dict(name=name, d=d, n=n, X=X, W=W, L1=L1, L2=L2))
    return ids, out


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event reasons during the timed region.  nvidia-smi -lms 100 runs as the
    profiling recipe's clocks line; an NVML thread samples every 5 ms so the short timed regions
    get enough samples.  mark() brackets the timed region; the summary uses the NVML samples
    inside it (else every sample)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.nv = []                      # (t, sm_mhz, reasons bitmask)
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self.handle = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(gpu_index)
            try:
                bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.nvml = pynvml
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.handle = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        if self.handle is not None:
            self.nth = threading.Thread(target=self._nvml, daemon=True)
            self.nth.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def _nvml(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle))
                self.nv.append((time.time(), mhz, rs))
            except Exception:
                return
            time.sleep(0.005)

    def mark(self, begin: bool):
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        self._stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if self.nv:
            nv = self.nvml
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            sel = [x for x in self.nv if self.t0 is not None and self.t1 is not None and self.t0 <= x[0] <= self.t1]
            inside = bool(sel)
            sel = sel or self.nv
            sm = [x[1] for x in sel]
            reasons = sorted(nm for nm, b in bits.items() if any(x[2] & b for x in sel))
            return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(sm), "source": "NVML every 5 ms" +
                    (" inside the timed region" if inside else " (whole run)"),
                    "nvidia_smi_samples": len(self.lines)}
        if self.proc is None:
            return None
        sm, mx, reasons = [], 0.0, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi -lms 100"}


# --------------------------------------------------------------------------- oracle arm
def oracle_sample_step(ids_s, lin_s, r):
    """The CPU oracle's step on a bounded sample (one linear, a few tokens): every §8(a) row."""
    import oracle as O
    X, W = lin_s["X"], lin_s["W"]
    R, cnt = O.calibrate_stats(X, ids_s, N_MOD)
    s = O.init_factors(R, cnt, W)
    qw, dw = O.quantize_weight(W, s[0], WBITS)
    L1 = list(lin_s["L1"]) if r > 0 else None
    L2 = list(lin_s["L2"]) if r > 0 else None
    O.linear_forward(X, ids_s, s, qw, dw, ABITS, L1, L2)
    O.calib_loss(X, ids_s, s, W, WBITS, ABITS)


def oracle_sample(T, r, seed_rank=0):
    """Sample = the qkv linear of the layer on k tokens of every modality (two sizes split the
    per-token from the per-step weight-side cost)."""
    cfg = synth.CONFIGS[CFG]
    name, d, n = layer_linears(["qkv"])[0]
    ids_full = synth.modality_ids(cfg["pattern"], T=T)
    X = synth.activations(ids_full, d, N_MOD, synth.seed_for(CI, 0, 0) + 100000 * seed_rank)
    W = synth.weight(d, n, synth.seed_for(CI, 0, 1))
    L1, L2 = synth.lowrank(d, n, r, N_MOD, synth.seed_for(CI, 0, 2)) if r > 0 else (None, None)
    by_mod = [np.nonzero(ids_full == m)[0] for m in range(N_MOD)]

    def sample(k):
        rows = np.concatenate([b[:k] for b in by_mod])
        return ids_full[rows], dict(X=X[rows], W=W, L1=L1, L2=L2)
    return sample


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def time_oracle(T, r, linears, repeats=4, k_small=128, k_large=512):
    """Returns (tokens/s extrapolated to the full layer at T tokens, seconds of CPU work, desc).
    ~10-15 s of oracle work: `repeats` steps at 2*k_small and at 2*k_large tokens."""
    sample = oracle_sample(T, r)
    ids_a, s_a = sample(k_small)
    ids_b, s_b = sample(k_large)
    t0 = time.perf_counter()
    oracle_sample_step(ids_a, s_a, r)                     # warm caches / BLAS threads
    t = time.perf_counter()
    for _ in range(repeats):
        oracle_sample_step(ids_a, s_a, r)
    ta = (time.perf_counter() - t) / repeats
    t = time.perf_counter()
    for _ in range(repeats):
        oracle_sample_step(ids_b, s_b, r)
    tb = (time.perf_counter() - t) / repeats
    total = time.perf_counter() - t0
    na, nb = N_MOD * k_small, N_MOD * k_large
    per_tok = max(tb - ta, 1e-9) / (nb - na)
    fixed = max(ta - na * per_tok, 0.0)
    _, dq, nq = layer_linears(["qkv"])[0]
    dn_qkv = dq * nq
    scale = sum(d * n for _, d, n in linears) / dn_qkv
    layer_time = scale * (fixed + T * per_tok)
    desc = (f"oracle step (stats, init, wquant, forward+CMC, loss incl. X W) on the qkv linear "
            f"{dq}->{nq} with {na} and {nb} tokens (equal shares of the {N_MOD} modalities), {repeats} repeats each: "
            f"{ta:.2f} s / {tb:.2f} s per step; extrapolated to the {len(linears)}-linear layer at {T} tokens "
            f"by sum(d*n) (x{scale:.1f}): {layer_time:.1f} s")
    return T / layer_time, total, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    linears = layer_linears(args.linears.split(","))
    T = args.tokens
    sample = oracle_sample(T, args.rank_cmc)
    ids32, s32 = sample(32)
    for _ in range(args.warmup):
        oracle_sample_step(ids32, s32, args.rank_cmc)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle_sample_step(ids32, s32, args.rank_cmc)
    step_s = (time.perf_counter() - t) / max(args.steps, 1)
    value, _, desc = time_oracle(T, args.rank_cmc, linears)
    cores = oracle_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": workload_config(args, linears),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, linears):
    if CFG == "c2":
        head = "c2 (BASELINE configs[1]): Qwen2.5-Omni-3B-shaped (thinker) decoder layer, linears "
        lay = "4 x [text 64 | image 512 | audio 320 | text 128]"
        mods = "3 modalities (text/image/audio)"
    else:
        head = "c3 (BASELINE configs[2]): Qwen2.5-VL-7B-shaped decoder layer, linears "
        lay = "16 x [text 64 | image 768 | text 192]"
        mods = "2 modalities (text/image)"
    return {
        "workload": (head + ", ".join(f"{k} {d}->{n}" for k, d, n in linears)
                     + f"; {args.tokens} tokens/GPU per step ({lay}); "
                     f"W{WBITS}A{ABITS}; CMC rank {args.rank_cmc} for non-text tokens; {mods}"),
        "tokens_per_gpu": args.tokens,
        "parallelism": f"dp{args.gpus} (token-sharded calibration; replicated weights)",
        "l2": "inputs larger than L2 (each step streams >1 GB of activations/weights; no flush)",
        "streams": args.streams,
    }



# --------------------------------------------------------------------------- c4 calibration sweep
def run_c4(args):
    """BASELINE configs[3]: full 28-layer Qwen2.5-VL-7B-shaped calibration sweep, 16384 tokens per
    GPU (128 samples x 1024 tokens over 8 GPUs).  Per sweep: A1 stats of every layer input, ONE
    batched MAX/SUM exchange for all layers, then per layer: A2 init, X W once (the loss target of
    the batch), and 2 S-optimisation epochs (N1): loss + straight-through gradient
    (global counts, SUM-reduced) + log-space Adam on every linear, each followed by a SUM exchange.
    Inputs are generated on the device (same recipe distribution as synth/, seeded per layer and
    rank): host generation of 28 layers would take minutes; parity is covered at c3 sizes."""
    import torch
    import torch.distributed as dist

    import paper_2603_04800_b200 as M
    from paper_2603_04800_b200 import parallel as P
    from paper_2603_04800_b200._lib import lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MASQ_BENCH_FUNCTIONAL=1: exercise the N>1 code path on one GPU (every rank on cuda:0, gloo
    # exchanges through the host) — a functional check of the multi-rank logic, never a timing
    functional = os.environ.get("MASQ_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    T = args.tokens
    linears = layer_linears(args.linears.split(","))
    ids_h = synth.modality_ids(synth.CONFIGS[CFG]["pattern"], T=T)
    ids = torch.from_numpy(ids_h).to(dev)
    g = torch.Generator(device=dev)
    layers = []
    for l in range(args.layers):
        g.manual_seed(synth.seed_for(3, l, 0) + 100000 * rank)
        ent = []
        for (name, d, n) in linears:
            chan = torch.exp(torch.randn(N_MOD, d, generator=g, device=dev))
            chan[:, torch.randperm(d, generator=g, device=dev)[: max(1, d // 100)]] *= 10.0
            scale = torch.tensor([1.0, 20.0], device=dev)[:, None] * chan
            X = (torch.randn(T, d, generator=g, device=dev) * scale[ids.long()]).to(torch.bfloat16)
            W = (torch.randn(d, n, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16)
            ent.append(dict(name=name, d=d, n=n, X=X, W=W))
        layers.append(ent)
    nl = len(linears)
    Rbuf = torch.zeros(args.layers * sum(N_MOD * e["d"] for e in layers[0]), dtype=torch.float32, device=dev)
    Rv, off = [], 0
    for l in range(args.layers):
        for e in layers[l]:
            Rv.append(Rbuf[off:off + N_MOD * e["d"]].view(N_MOD, e["d"]))
            off += N_MOD * e["d"]
    Cbuf = torch.zeros(args.layers * nl, N_MOD, dtype=torch.int64, device=dev)
    Yref = [torch.empty(T, e["n"], dtype=torch.float32, device=dev) for e in layers[0]]
    Sbuf = torch.zeros(nl, N_MOD, dtype=torch.float64, device=dev)
    Nbuf = torch.zeros(nl, N_MOD, dtype=torch.int64, device=dev)
    losses = torch.zeros(args.layers, 2, nl, dtype=torch.float64, device=dev)
    ws = M.Workspace(dev)
    # linear li of a layer runs on stream li % S with its own workspace (the linears of a layer are
    # independent between the exchanges; 2 streams let one linear's HBM-bound kernels run beside
    # another's GEMM)
    nstreams = max(1, args.streams)
    main = torch.cuda.current_stream()
    side = [torch.cuda.Stream(device=dev) for _ in range(nstreams)] if nstreams > 1 else []
    wss = [ws] + [M.Workspace(dev) for _ in range(nstreams - 1)]

    def on(li):
        return torch.cuda.stream(side[li % nstreams]) if side else contextlib.nullcontext()

    def fork():
        if side:
            ev = torch.cuda.Event()
            ev.record(main)
            for st_ in side:
                st_.wait_event(ev)

    def join():
        for st_ in side:
            main.wait_stream(st_)

    # every loss pass is a real S-optimisation step (N1): loss + straight-through gradient + Adam
    optimise = True
    grads = [torch.empty(N_MOD, e["d"], dtype=torch.float64, device=dev) for e in layers[0]]
    adam = [None] * nl

    def sweep():
        for l in range(args.layers):
            for li, e in enumerate(layers[l]):
                M.calibrate_stats(e["X"], ids, N_MOD, R=Rv[l * nl + li], count=Cbuf[l * nl + li], reset=True, ws=ws)
        P.reduce_stats([Rbuf], Cbuf)
        for l in range(args.layers):
            fork()
            svec = [None] * nl
            for li, e in enumerate(layers[l]):
                with on(li):
                    wk = wss[li % nstreams]
                    svec[li] = M.init_factors(Rv[l * nl + li], Cbuf[l * nl + li], e["W"], ws=wk)
                    M.reference_output(e["X"], e["W"], Yref=Yref[li], ws=wk)
                    if optimise:
                        adam[li] = M.adam_init(svec[li])
            for p_ in range(2):
                for li, e in enumerate(layers[l]):
                    with on(li):
                        wk = wss[li % nstreams]
                        # N1: 2 epochs of loss + straight-through gradient + log-space
                        # Adam, the gradient normalised by the global counts and SUM-reduced
                        M.calib_loss_grad(e["X"], ids, svec[li], e["W"], WBITS, ABITS, Yref[li], grad=grads[li],
                                          sums=Sbuf[li], counts=Nbuf[li], loss=losses[l, p_, li:li + 1],
                                          count_norm=Cbuf[l * nl + li], ws=wk)
                if world > 1:
                    join()
                    P.reduce_loss(Sbuf, Nbuf)
                    for li, e in enumerate(layers[l]):
                        if optimise:
                            P.reduce_grad(grads[li])
                        M.loss_finalize(Sbuf[li], Nbuf[li], e["n"], loss=losses[l, p_, li:li + 1])
                    fork()
                if optimise:
                    for li, e in enumerate(layers[l]):
                        with on(li):
                            th, m1, m2 = adam[li]
                            M.adam_step(th, grads[li], m1, m2, p_ + 1, 1e-2, s_out=svec[li])
            join()

    # the clock sampler starts before the warm-up, so no idle gap precedes the timed region
    clk = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if clk:
        clk.start()
    for _ in range(max(args.warmup, 1)):
        sweep()
    for w in wss:
        M.check(w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lib().masq_profile_enable(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clk:
        clk.mark(True)
    a.record()
    for _ in range(args.steps):
        sweep()
    b.record()
    torch.cuda.synchronize()
    if clk:
        clk.mark(False)
    if world > 1:
        dist.barrier()
    clocks = clk.stop() if clk else None
    import ctypes
    names = ctypes.create_string_buffer(32 * 64)
    tot = (ctypes.c_double * 64)()
    cnt = (ctypes.c_int64 * 64)()
    nk = lib().masq_profile_collect(64, names, tot, cnt)
    lib().masq_profile_enable(0)
    kern = {names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): dict(ms_per_sweep=tot[i] / args.steps,
            launches_per_sweep=cnt[i] / args.steps) for i in range(max(nk, 0))}
    ms = P.max_over_ranks(a.elapsed_time(b), device=dev)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": world * T * args.steps / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic (device-generated, seeded)",
            "config": {"workload": (f"c4 (BASELINE configs[3]): {args.layers}-layer Qwen2.5-VL-7B-shaped calibration "
                                    f"sweep, {T} tokens/GPU (16 x [text 64 | image 768 | text 192]), per layer: stats "
                                    "of 4 inputs, init, X W once, "
                                    + ("2 S-optimisation epochs (loss + straight-through gradient + Adam, N1)"
                                       if optimise else "2 loss passes")
                                    + " (W4A8); one MAX/SUM exchange for all layers' stats, one SUM per pass"),
                       "tokens_per_gpu": T, "parallelism": f"dp{world}"},
            "kernels": kern, "gpu_launches": int(sum(v["launches_per_sweep"] for v in kern.values()) * args.steps),
            "clocks": clocks, "losses_layer0": [float(x) for x in losses[0].flatten().cpu().tolist()]}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0

def run_c5(args):
    """BASELINE configs[4]: masq_linear_forward at d = 3584 on --tokens mixed-modality tokens (c3
    span layout), W4A8, CMC rank --rank-cmc, output channels --c5-n.  With N ranks the forward is
    column-sharded: X, ids and the factors are replicated, rank g quantizes and owns
    columns parallel.column_shards(n, N)[g] of W (codes, scales, L2) and writes Y[:, shard]; no
    collective in the timed region (the caller gathers Y if it needs it whole).  `value` is the
    whole job's TOP/s (2 T d n over the max-over-ranks time: strong scaling, fixed total work).
    Weight quantization is inference-time preparation and sits outside the timed region."""
    import torch
    import torch.distributed as dist

    import paper_2603_04800_b200 as M
    from paper_2603_04800_b200 import parallel as P
    from paper_2603_04800_b200._lib import lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("MASQ_BENCH_FUNCTIONAL") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if os.environ.get("MASQ_BENCH_FUNCTIONAL") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    T, d, n, r = args.tokens, 3584, args.c5_n, args.rank_cmc
    g = torch.Generator(device=dev)
    g.manual_seed(synth.seed_for(4, 0, 0))                  # same inputs on every rank (replicated X)
    ids_h = synth.modality_ids(synth.CONFIGS[CFG]["pattern"], T=T)
    ids = torch.from_numpy(ids_h).to(dev)
    chan = torch.exp(torch.randn(N_MOD, d, generator=g, device=dev))
    chan[:, torch.randperm(d, generator=g, device=dev)[: max(1, d // 100)]] *= 10.0
    scale = torch.tensor([1.0, 20.0], device=dev)[:, None] * chan
    X = (torch.randn(T, d, generator=g, device=dev) * scale[ids.long()]).to(torch.bfloat16)
    W = (torch.randn(d, n, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16)
    L1 = (torch.randn(N_MOD - 1, d, r, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16) if r else None
    L2 = (torch.randn(N_MOD - 1, r, n, generator=g, device=dev) * (4.0 / r ** 0.5)).to(torch.bfloat16) if r else None
    R, cnt = M.calibrate_stats(X, ids, N_MOD)
    s = M.init_factors(R, cnt, W)
    j0, j1 = P.column_shards(n, world)[rank]
    qw, dw = M.quantize_weight(W[:, j0:j1].contiguous(), s[0], WBITS)
    L2s = L2[:, :, j0:j1] if r else None                   # column view, row stride n
    Y = torch.empty(T, j1 - j0, dtype=torch.float32, device=dev)
    ws = M.Workspace(dev)

    def fwd():
        M.linear_forward(X, ids, s, qw, dw, WBITS, ABITS, L1, L2s, Y=Y, ws=ws)

    clk = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if clk:
        clk.start()                      # before the warm-up: no idle gap before the timed region
    for _ in range(max(args.warmup, 1)):
        fwd()
    M.check(ws)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lib().masq_profile_enable(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clk:
        clk.mark(True)
    a.record()
    for _ in range(args.steps):
        fwd()
    b.record()
    torch.cuda.synchronize()
    if clk:
        clk.mark(False)
    if world > 1:
        dist.barrier()
    clocks = clk.stop() if clk else None
    import ctypes
    names = ctypes.create_string_buffer(32 * 64)
    tot = (ctypes.c_double * 64)()
    cntk = (ctypes.c_int64 * 64)()
    nk = lib().masq_profile_collect(64, names, tot, cntk)
    lib().masq_profile_enable(0)
    kern = {names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): dict(ms_per_call=tot[i] / args.steps,
            launches_per_call=cntk[i] / args.steps) for i in range(max(nk, 0))}
    ms = P.max_over_ranks(a.elapsed_time(b), device=dev) / args.steps
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops_sustained": 1412.5}
    int8_peak = 2.0 * float(pk["bf16_tflops_sustained"]) * world
    ops = 2.0 * T * d * n
    value = ops / (ms / 1e3) / 1e12
    gk = kern.get("gemm_fwd", {}).get("ms_per_call")
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "TOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int8", "data": "synthetic (device-generated, seeded)",
            "config": {"workload": f"c5 (BASELINE configs[4]): masq_linear_forward, {T} mixed-modality tokens "
                                   f"(16 x [text 64 | image 768 | text 192] layout), d 3584 -> {n}, W4A8, CMC rank "
                                   f"{r}; output columns sharded over {world} GPU(s)",
                       "tokens": T, "d": d, "n": n, "parallelism": f"column-shard x{world}"},
            "roofline": {"bound": "tensor", "achieved": value, "peak": int8_peak, "unit": "TOP/s",
                         "frac": value / int8_peak, "scope": "whole masq_linear_forward call, all ranks",
                         "peak_source": "MEASURED_PEAKS.json bf16 sustained x 2 (INT8/bf16 nominal ratio) x ranks",
                         "gemm_kernel_tops": (ops / world) / (gk / 1e3) / 1e12 if gk else None},
            "kernels": kern, "clocks": clocks,
            "functional_check": os.environ.get("MASQ_BENCH_FUNCTIONAL") == "1"}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- GPU arm
ROOFLINE_KERNEL = "gemm_ref"           # the step's dominant kernel (X W, ~43% of the c3 step)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload in ("c4", "c4s"):
        return run_c4(args)
    if args.workload == "c5":
        return run_c5(args)

    import torch
    import torch.distributed as dist

    import paper_2603_04800_b200 as M
    from paper_2603_04800_b200 import parallel as P
    from paper_2603_04800_b200._lib import lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MASQ_BENCH_FUNCTIONAL=1: exercise the N>1 code path on one GPU (every rank on cuda:0, gloo
    # exchanges through the host) — a functional check of the multi-rank logic, never a timing
    functional = os.environ.get("MASQ_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    linears = layer_linears(args.linears.split(","))
    T, r = args.tokens, args.rank_cmc
    ids_h, lins_h = make_host_inputs(T, rank, linears, r)

    def to_dev_bf16(a):
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(dev)

    ids = torch.from_numpy(ids_h).to(dev)
    L = []
    for lh in lins_h:
        d, n = lh["d"], lh["n"]
        e = dict(name=lh["name"], d=d, n=n, X=to_dev_bf16(lh["X"]), W=to_dev_bf16(lh["W"]),
                 L1=to_dev_bf16(lh["L1"]) if r > 0 else None, L2=to_dev_bf16(lh["L2"]) if r > 0 else None,
                 Y=torch.empty(T, n, dtype=torch.float32, device=dev),
                 Yref=torch.empty(T, n, dtype=torch.float32, device=dev),
                 Xpin=torch.from_numpy(lh["X"].view(np.int16)).view(torch.bfloat16).pin_memory())
        L.append(e)
    ids_pin = torch.from_numpy(ids_h).pin_memory()
    nl = len(L)
    Rbuf = torch.zeros(sum(N_MOD * e["d"] for e in L), dtype=torch.float32, device=dev)   # one flat buffer
    Rv, off = [], 0
    for e in L:                                          # contiguous [N_MOD x d] views (ABI layout)
        Rv.append(Rbuf[off:off + N_MOD * e["d"]].view(N_MOD, e["d"]))
        off += N_MOD * e["d"]
    Cbuf = torch.zeros(nl, N_MOD, dtype=torch.int64, device=dev)
    Sbuf = torch.zeros(nl, N_MOD, dtype=torch.float64, device=dev)
    Nbuf = torch.zeros(nl, N_MOD, dtype=torch.int64, device=dev)
    losses = torch.zeros(nl, dtype=torch.float64, device=dev)
    ws = M.Workspace(dev)

    nside = max(2, args.streams)
    side_all = [torch.cuda.Stream(device=dev) for _ in range(nside)]
    wss = [ws] + [M.Workspace(dev) for _ in range(nside - 1)]

    nvtx_on = bool(getattr(args, "nvtx", False))

    def rng(name):
        if nvtx_on:
            torch.cuda.nvtx.range_push(name)

    def rng_end():
        if nvtx_on:
            torch.cuda.nvtx.range_pop()

    def step(X_override=None, ids_override=None, nstreams=None):
        nstreams = max(1, args.streams if nstreams is None else nstreams)
        side = side_all[:nstreams] if nstreams > 1 else []
        idt = ids if ids_override is None else ids_override
        rng("A1 stats + exchange")
        for li, e in enumerate(L):
            X = e["X"] if X_override is None else X_override[li]
            M.calibrate_stats(X, idt, N_MOD, R=Rv[li], count=Cbuf[li], reset=True, ws=ws)
        P.reduce_stats([Rbuf], Cbuf)                    # one batched exchange per step (max is order-free)
        rng_end()
        main = torch.cuda.current_stream()
        if side:
            ready = torch.cuda.Event()
            ready.record(main)
        for li, e in enumerate(L):
            X = e["X"] if X_override is None else X_override[li]
            k = li % nstreams
            if side:
                side[k].wait_event(ready)
            with torch.cuda.stream(side[k] if side else main):
                rng(f"linear {e['name']} (A2-A8)")
                s = M.init_factors(Rv[li], Cbuf[li], e["W"], ws=wss[k])
                e["s"] = s
                # A3 (every modality's weight codes, one W read) + A4-A7 forward + A8 target and loss
                M.calib_layer(X, idt, s, e["W"], WBITS, ABITS, e["L1"], e["L2"], Y=e["Y"], Yref=e["Yref"],
                              sums=Sbuf[li], counts=Nbuf[li], loss=losses[li:li + 1], ws=wss[k])
                rng_end()
        for st_ in side:                                 # join before the exchange / the step's end
            main.wait_stream(st_)
        if world > 1:
            P.reduce_loss(Sbuf, Nbuf)
            for li, e in enumerate(L):
                M.loss_finalize(Sbuf[li], Nbuf[li], e["n"], loss=losses[li:li + 1])

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        return P.max_over_ranks(x, device=dev)

    # ------------------------------------------------------------------ warm-up
    # the clock sampler starts before the warm-up, so no idle gap (a sleep for the sampler thread
    # had let the GPU's power budget recover) precedes the timed region: the timed steps follow
    # the warm-up steps at the sustained, power-capped operating point
    clk = ClockSampler(torch.cuda.current_device()) if rank == 0 and not args.profile_only else None
    if clk:
        clk.start()
    for _ in range(max(args.warmup, 0)):
        step()
    for w in wss:
        M.check(w)
    torch.cuda.synchronize()

    if args.profile_only:
        step()
        torch.cuda.synchronize()
        print(json.dumps({"profile_only": True, "loss": losses.tolist()}), flush=True)
        return 0

    # ------------------------------------------------------------------ timed region (device)
    barrier()
    torch.cuda.synchronize()
    # --graph (N=1): the whole layer step (64 library launches + memsets) is captured once as a
    # CUDA graph and replayed; the library's profiler events are captured with it as external
    # event nodes, so every replay re-times the kernels and the breakdown below is that of the
    # last timed replay.  Default: eager launches (kernels cover ~98% of the step already).
    use_graph = world == 1 and args.graph
    graph = None
    # Eager (default): inside the timed region the library's profiler brackets ONLY the X W GEMM
    # launches (the dominant kernel, whose CUDA-event durations the roofline needs); every other
    # kernel runs between unbracketed neighbours, so the programmatic dependent launches overlap
    # as they do for a user.  The per-kernel table comes from a breakdown pass of the same K
    # steps right after, with every kernel bracketed.
    if use_graph:
        lib().masq_profile_enable(1)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
    else:
        lib().masq_profile_only(ROOFLINE_KERNEL.encode())
        lib().masq_profile_enable(1)
    prof_steps = 1 if use_graph else args.steps
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
    if clk:
        clk.mark(True)
    ev0.record()
    for k_ in range(args.steps):
        if use_graph:
            graph.replay()
        else:
            step()
        if k_ < args.steps - 1:
            evs[k_].record()
    ev1.record()
    torch.cuda.synchronize()
    if clk:
        clk.mark(False)
    barrier()
    clocks = clk.stop() if clk else None
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    marks = [ev0] + evs + [ev1]
    ms_median = float(np.median([marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]))
    import ctypes

    def collect_kernels():
        cap = 64
        names = ctypes.create_string_buffer(32 * cap)
        tot = (ctypes.c_double * cap)()
        cnt = (ctypes.c_int64 * cap)()
        nk = lib().masq_profile_collect(cap, names, tot, cnt)
        out = {}
        for i in range(max(nk, 0)):
            nm = names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode()
            out[nm] = dict(ms=tot[i], launches=int(cnt[i]))
        return out

    kern_timed = collect_kernels()
    lib().masq_profile_enable(0)
    lib().masq_profile_only(None)
    for w in wss:
        M.check(w)
    ms_step = ms_total / args.steps
    value = world * T * args.steps / (ms_total / 1e3)

    # ------------------------------------------------------------------ per-kernel breakdown
    kern, ms_bd = kern_timed, ms_step
    if not use_graph:
        torch.cuda.synchronize()
        barrier()
        lib().masq_profile_enable(1)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record()
        for _ in range(args.steps):
            step()
        b1.record()
        torch.cuda.synchronize()
        kern = collect_kernels()
        lib().masq_profile_enable(0)
        ms_bd = b0.elapsed_time(b1) / args.steps
        barrier()

    # ------------------------------------------------------------------ unprofiled (1 stream)
    # The same K steps again with no event records at all (the timed region above still brackets
    # the X W launches for the roofline; an event record between two kernels serialises them).
    unprofiled = None
    if args.streams == 1:
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        u0.record()
        for _ in range(args.steps):
            step()
        u1.record()
        torch.cuda.synchronize()
        barrier()
        ms_u = max_over_ranks(u0.elapsed_time(u1))
        unprofiled = {"streams": 1, "ms_per_step": ms_u / args.steps,
                      "value": world * T * args.steps / (ms_u / 1e3), "unit": "tokens/s",
                      "pdl": os.environ.get("MASQ_PDL", "1") != "0",
                      "note": "same step, same stream, no event records at all (the timed region brackets only the "
                              "X W launches); run after the breakdown pass, so the GPU's power / thermal state "
                              "differs from the timed region's"}

    # ------------------------------------------------------------------ overlapped (2 streams)
    # The same step with the linears on 2 CUDA streams (one linear's HBM-bound kernels beside
    # another's GEMM), timed separately so the per-kernel CUDA-event durations above stay clean.
    overlapped = None
    if args.streams == 1:
        for _ in range(2):
            step(nstreams=2)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        o0, o1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        o0.record()
        for _ in range(args.steps):
            step(nstreams=2)
        o1.record()
        torch.cuda.synchronize()
        barrier()
        ms_o = max_over_ranks(o0.elapsed_time(o1))
        overlapped = {"streams": 2, "ms_per_step": ms_o / args.steps,
                      "value": world * T * args.steps / (ms_o / 1e3), "unit": "tokens/s",
                      "note": "same step, the 4 linears spread over 2 CUDA streams (per-stream workspaces); "
                              "timed after the main region, no profiler"}

    # ------------------------------------------------------------------ e2e (host buffers)
    # Every step copies its inputs (the layer's activations + modality ids) from pinned host
    # memory and reads the per-linear losses back.  The copies run on a second stream into a
    # double-buffered set of device inputs, so step k's H2D overlaps step k-1's compute.
    e2e = None
    if not args.no_e2e:
        xin = [[torch.empty_like(e["X"]) for e in L] for _ in range(2)]
        idin = [torch.empty_like(ids) for _ in range(2)]
        host_out = torch.empty(losses.numel(), dtype=torch.float64).pin_memory()
        h2d = sum(e["Xpin"].numel() * 2 for e in L) + ids_pin.numel()
        d2h = losses.numel() * 8
        comp = torch.cuda.current_stream()
        copy_s = torch.cuda.Stream()
        copied = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]

        def e2e_run(k_steps):
            for k in range(k_steps):
                b = k & 1
                with torch.cuda.stream(copy_s):
                    if k >= 2:
                        copy_s.wait_event(freed[b])
                    for li, e in enumerate(L):
                        xin[b][li].copy_(e["Xpin"], non_blocking=True)
                    idin[b].copy_(ids_pin, non_blocking=True)
                    copied[b].record(copy_s)
                comp.wait_event(copied[b])
                step(X_override=xin[b], ids_override=idin[b])
                freed[b].record(comp)
                host_out.copy_(losses, non_blocking=True)

        e2e_run(2)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(comp)
        copy_s.wait_stream(comp)
        e2e_run(args.steps)
        b_ev.record(comp)
        torch.cuda.synchronize()
        barrier()
        ms_e2e = max_over_ranks(a_ev.elapsed_time(b_ev))
        e2e = {"value": world * T * args.steps / (ms_e2e / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": ms_e2e / args.steps,
               "note": "pinned H2D of the step's activations+ids on a copy stream (double-buffered, overlapping "
                       "the previous step's compute) + D2H of the per-linear losses (the step's result), every "
                       "step; the forward outputs Y and the targets X W stay on the device (a calibration step "
                       "consumes them there)"}

    # ------------------------------------------------------------------ N1 (S-optimisation step)
    loss_main = [float(x) for x in losses.cpu().tolist()]
    n1 = None
    if not args.no_n1:
        for e in L:
            e["theta"], e["m1"], e["m2"] = M.adam_init(e["s"])
            e["grad"] = torch.empty_like(e["theta"])
        Gbuf = [e["grad"] for e in L]
        n1_state = {"t": 0}

        def n1_step():
            n1_state["t"] += 1
            for li, e in enumerate(L):
                M.calib_loss_grad(e["X"], ids, e["s"], e["W"], WBITS, ABITS, e["Yref"], grad=e["grad"],
                                  sums=Sbuf[li], counts=Nbuf[li], loss=losses[li:li + 1],
                                  count_norm=Cbuf[li], ws=ws)
            if world > 1:
                for g in Gbuf:
                    P.reduce_grad(g)
            for e in L:
                M.adam_step(e["theta"], e["grad"], e["m1"], e["m2"], n1_state["t"], 1e-3, s_out=e["s"])

        for _ in range(max(args.warmup, 0)):
            n1_step()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        # timed: only the gradient GEMM's launches bracketed (its roofline); then a breakdown pass
        lib().masq_profile_only(b"gradgemm")
        lib().masq_profile_enable(1)
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record()
        for _ in range(args.steps):
            n1_step()
        b_ev.record()
        torch.cuda.synchronize()
        barrier()
        ms_n1 = max_over_ranks(a_ev.elapsed_time(b_ev))
        kg = collect_kernels()
        lib().masq_profile_enable(0)
        lib().masq_profile_only(None)
        lib().masq_profile_enable(1)
        for _ in range(args.steps):
            n1_step()
        torch.cuda.synchronize()
        kn1 = collect_kernels()
        lib().masq_profile_enable(0)
        barrier()
        M.check(ws)
        k1 = {nm: v["ms"] for nm, v in kn1.items()}
        if "gradgemm" in kg:
            k1["gradgemm"] = kg["gradgemm"]["ms"]
        gg_ms = k1.get("gradgemm", 0.0) / args.steps
        gflop = sum(4.0 * T * e["d"] * e["n"] for e in L)
        peaks1 = load_peaks()
        n1 = {"ms_per_step": ms_n1 / args.steps,
              "tokens_per_s": world * T * args.steps / (ms_n1 / 1e3),
              "kernels_ms_per_step": {k: v / args.steps for k, v in k1.items()},
              "gradgemm": {"bound": "tensor", "flops_per_step": gflop,
                           "achieved": gflop / (gg_ms / 1e3) / 1e12 if gg_ms else None, "unit": "TFLOP/s",
                           "peak": peaks1["bf16"],
                           "frac": (gflop / (gg_ms / 1e3) / 1e12 / peaks1["bf16"]) if gg_ms else None,
                           "peak_source": "MEASURED_PEAKS.json bf16 burst"},
              "gpu_launches_per_step": sum(v["launches"] for v in kn1.values()) / args.steps,
              "losses_after": [float(x) for x in losses.cpu().tolist()],
              "note": "per linear: masq_calib_loss_grad (global-count normalised) -> NCCL SUM of grad (N>1) -> "
                      "masq_adam_step (lr 1e-3); outside the timed §8(a) step; only the gradient GEMM's launches carry "
                      "events while timing (gradgemm from there), the other kernels from a breakdown pass"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ------------------------------------------------------------------ INT8 ceiling, measured here
    # cuBLAS's int8 GEMM (torch._int_mm) on the step's largest linear shape, timed in this process
    # after the timed regions (a second, measured denominator beside the derived 2 x bf16 one)
    int8_ceiling = None
    try:
        big = max(L, key=lambda e: e["d"] * e["n"])
        a8 = torch.randint(-127, 128, (T, big["d"]), dtype=torch.int8, device=dev)
        b8 = torch.randint(-8, 8, (big["n"], big["d"]), dtype=torch.int8, device=dev).t()
        for _ in range(3):
            torch._int_mm(a8, b8)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        c0.record()
        for _ in range(reps):
            torch._int_mm(a8, b8)
        c1.record()
        torch.cuda.synchronize()
        ms_i = c0.elapsed_time(c1) / reps
        int8_ceiling = {"tops": 2.0 * T * big["d"] * big["n"] / (ms_i * 1e-3) / 1e12,
                        "shape": f"{T} x {big['d']} x {big['n']}", "ms": ms_i,
                        "how": "torch._int_mm (cuBLAS s8 GEMM), 10 back-to-back calls after 3 warm-up, CUDA events"}
        del a8, b8
    except Exception as ex:
        int8_ceiling = {"tops": None, "error": repr(ex)}

    # ------------------------------------------------------------------ roofline accounting
    peaks = load_peaks()
    int8_peak = 2.0 * peaks["bf16_sus"]          # INT8 = 2x bf16 (nominal ratio 4.5/2.25 PFLOP/s)
    bf16_peak = peaks["bf16_sus"]
    ops = sum(2.0 * T * e["d"] * e["n"] for e in L)                 # per step, one pass of all linears
    n_nt = int((ids_h != 0).sum())
    kinfo = {}
    K = prof_steps                                    # steps the per-kernel event totals cover
    per_step = {
        "gemm_fwd": ("tensor", ops, "TOP/s", int8_peak),
        # text rows' loss comes out of the forward's epilogue (S_0 = S_t); the loss GEMM runs on the
        # non-text rows only
        "gemm_loss": ("tensor", sum(2.0 * n_nt * e["d"] * e["n"] for e in L), "TOP/s", int8_peak),
        "gemm_ref": ("tensor", ops, "TFLOP/s", bf16_peak),
        "stats": ("hbm", sum(2.0 * T * e["d"] + T for e in L), "GB/s", peaks["hbm"]),
        # X read (2 B) + token-order codes (1 B) + the modality-grouped copy of the non-text rows
        # (1 B, masq_calib_layer's loss operand) per activation, + the row scales
        "aquant": ("hbm", sum(3.0 * T * e["d"] + 1.0 * n_nt * e["d"] + 4 * T + 4 * n_nt for e in L), "GB/s",
                   peaks["hbm"]),
        "gather_rows": ("hbm", sum(2.0 * T * e["d"] for e in L), "GB/s", peaks["hbm"]),
        # X rows of the non-text tokens (2 B) + their Z row: (M-1) modalities x [hi | lo] x rpad bf16
        "zgemm": ("hbm", sum(2.0 * n_nt * e["d"] + 2.0 * n_nt * (N_MOD - 1) * 2 * (-(-max(r, 1) // 64) * 64)
                             for e in L), "GB/s", peaks["hbm"]),
        "wcolmax": ("hbm", sum(2.0 * e["d"] * e["n"] for e in L), "GB/s", peaks["hbm"]),      # one W read, N_MOD sets
        "wquant": ("hbm", sum((2.0 + N_MOD) * e["d"] * e["n"] for e in L), "GB/s", peaks["hbm"]),
        "init": ("hbm", sum(2.0 * e["d"] * e["n"] for e in L), "GB/s", peaks["hbm"]),
    }
    total_kernel_ms = sum(v["ms"] for v in kern.values())
    for nm, v in kern.items():
        ent = {"ms_per_step": v["ms"] / K, "launches_per_step": v["launches"] / K,
               "share_of_step": (v["ms"] / K) / ms_bd}
        if nm in per_step:
            bound, work, unit, peak = per_step[nm]
            ach = work / (v["ms"] / K / 1e3) / (1e12 if unit != "GB/s" else 1e9)
            ent.update(bound=bound, achieved=ach, unit=unit, peak=peak, frac=ach / peak)
        kinfo[nm] = ent
    dom = max(kern, key=lambda k: kern[k]["ms"]) if kern else None
    traffic = None
    # DRAM bytes per launch from an ncu capture of THIS workload's step (c3: ncu_traffic.json;
    # others: ncu_traffic_<workload>.json), else null
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json" if args.workload == "c3"
                      else f"ncu_traffic_{args.workload}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom)
        except Exception:
            traffic = None
    roof = None
    if dom and "achieved" in kinfo.get(dom, {}):
        k = kinfo[dom]
        # the dominant kernel's durations from the timed region itself (its launches are the
        # ones bracketed there); the breakdown pass's value as a fallback
        src = kern_timed if dom in kern_timed else kern
        bound, work, unit, peak = per_step[dom]
        ach = work / (src[dom]["ms"] / prof_steps / 1e3) / (1e12 if unit != "GB/s" else 1e9)
        roof = {"kernel": dom, "bound": bound, "achieved": ach, "peak": peak,
                "unit": unit, "frac": ach / peak, "traffic": traffic,
                "peak_source": f"{peaks['src']} MEASURED_PEAKS.json bf16 sustained"
                               + (" x2 (INT8/bf16 nominal ratio)" if dom != "gemm_ref" else ""),
                "avg_launch_ms": src[dom]["ms"] / src[dom]["launches"],
                "events": "timed region" if src is kern_timed else "breakdown pass",
                "share_of_step": (src[dom]["ms"] / prof_steps) / ms_step}
    fwd = kinfo.get("gemm_fwd", {})
    fwd_call_ms = sum(kinfo.get(k, {}).get("ms_per_step", 0.0) for k in ("inv", "aquant", "transpose", "l1_fold", "cmc_pack",
                                                                          "zgemm", "gemm_fwd"))
    linear = {
        "tops_gemm_kernel": fwd.get("achieved"),
        "frac_int8_peak_gemm_kernel": fwd.get("frac"),
        "tops_linear_forward_call": ops / (fwd_call_ms / 1e3) / 1e12 if fwd_call_ms else None,
        "frac_int8_peak_linear_forward_call": (ops / (fwd_call_ms / 1e3) / 1e12 / int8_peak) if fwd_call_ms else None,
        "frac_int8_spec_4500": (ops / (fwd_call_ms / 1e3) / 1e12 / 4500.0) if fwd_call_ms else None,
        "int8_peak_tops": int8_peak,
        "int8_peak_source": "MEASURED_PEAKS.json bf16 sustained x 2 (the guide's INT8/bf16 nominal ratio)",
        "frac_int8_spec_4500_gemm_kernel": (fwd.get("achieved") / 4500.0) if fwd.get("achieved") else None,
        "int8_ceiling_cublas": int8_ceiling,
        "frac_int8_ceiling_cublas_gemm_kernel": (fwd.get("achieved") / int8_ceiling["tops"])
        if (fwd.get("achieved") and int8_ceiling and int8_ceiling.get("tops")) else None,
        "note": "algorithmic 2*T*d*n ops of the 4 linears; forward = inv + aquant + L1/L2 pack (cmc_pack) + zgemm + gemm_fwd "
                "(the activation codes are computed once per step and shared with the loss)",
    }
    launches = int(sum(v["launches"] for v in kern.values())) * (args.steps // K)   # over the timed region

    cpu = None
    if not args.no_cpu_baseline and world >= 1 and rank == 0 and args.gpus == 1:
        try:
            v, secs, desc = time_oracle(T, r, linears)
            cpu = {"value": v, "unit": "tokens/s", "cores": oracle_threads(), "kind": "oracle", "sample": desc,
                   "seconds": secs}
            try:                                    # the same sample on ONE host thread
                from threadpoolctl import threadpool_limits
                with threadpool_limits(limits=1):
                    v1, secs1, _ = time_oracle(T, r, linears, repeats=2)
                cpu["value_1thread"] = v1
                cpu["seconds_1thread"] = secs1
            except Exception as ex:
                cpu["value_1thread"] = None
                cpu["error_1thread"] = repr(ex)
        except Exception as ex:  # report, never hide
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {ex!r}"}

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int8",
        "dtype_detail": f"s8 x s8 -> s32 tcgen05 GEMMs (W{WBITS}A{ABITS} codes in int8 containers); f32 quantizer; "
                        "bf16 -> f32 tcgen05 for CMC and X W",
        "data": "synthetic (seeded, synth/; random-init weights of the "
                + ("Qwen2.5-Omni-3B" if CFG == "c2" else "Qwen2.5-VL-7B") + " layer shapes)",
        "ms_per_step_median": ms_median,
        "config": workload_config(args, linears),
        "linear_forward": linear,
        "n1_s_opt_step": n1,
        "roofline": roof,
        "kernels": kinfo,
        "kernel_ms_sum_over_step_ms": (total_kernel_ms / K) / ms_bd if ms_bd else None,
        "kernels_source": ("breakdown pass: the same K steps right after the timed region, every library kernel "
                           f"bracketed by a CUDA-event pair ({ms_bd:.3f} ms/step there)") if not use_graph
                          else "the last timed graph replay",
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "cuda_graph": use_graph,
        "clocks": clocks,
        "e2e": e2e,
        "unprofiled": unprofiled,
        "overlapped": overlapped,
        "cpu_baseline": cpu,
        "losses": loss_main,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
