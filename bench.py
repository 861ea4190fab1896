#!/usr/bin/env python
"""Benchmark: windowed secure ReLU layer throughput (elements/s) on B200.

Workload (BASELINE.json configs[1] at the north-star size): one ReLU layer of
n = 2^24 fixed-point elements (x_f ~ N(0, 4^2), f = 16, N = 64), window
(k, m) = (22, 14), i.e. the 8-bit reduced ring.  A step = both parties of one
party pair evaluating the whole protocol (L+3 = 6 rounds) on the layer.

  N = 1   one party pair time-sliced on the GPU: the fused pair kernel
          (hb_relu_pair), openings exchanged through shared memory.
  N > 1   (torchrun) ranks 2i / 2i+1 are parties 0 / 1 of pair i, each pair on
          its own batch shard (weak scaling); every round is an NCCL
          send/recv between the two ranks (staged driver, hb_relu_round).

Prints ONE JSON line on rank 0.  `--impl reference` times the reference
algorithm on the host instead (the oracle port, see oracle/hb_oracle.py).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "secure_relu_elems_per_s"
UNIT = "elements/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--logn", type=int, default=24)
    p.add_argument("--k", type=int, default=22)
    p.add_argument("--m", type=int, default=14)
    p.add_argument("--ring-bits", type=int, default=64)
    p.add_argument("--path", choices=["pair", "staged", "p2p"], default="pair",
                   help="N=1 driver: fused pair kernel, staged rounds, or the P2P party kernels on two streams")
    p.add_argument("--p2p-scope", choices=["gpu", "sys"], default="gpu",
                   help="--path p2p: flag scope of the one-device harness (gpu = the scope both parties share; "
                        "sys = the cross-GPU protocol)")
    p.add_argument("--multi-path", choices=["p2p", "nccl"], default="p2p",
                   help="N>1: one-launch NVLink party kernel (peer buffers over CUDA IPC) or staged rounds + NCCL")
    p.add_argument("--graph", action="store_true",
                   help="capture the timed steps in one CUDA graph (no host launch overhead; small layers)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-resnet", action="store_true", help="skip the ResNet18 secondary measurement")
    p.add_argument("--sweep", default=None, help="write a (n, w) sweep table to this JSON file")
    p.add_argument("--triple-gb", type=float, default=64.0, help="HBM budget for stocked triples")
    p.add_argument("--workload", choices=["relu", "resnet18", "resnet50"], default="relu")
    p.add_argument("--batch", type=int, default=None, help="ResNet batch (default 512 / 128)")
    p.add_argument("--relu-config", default="search",
                   help="ResNet per-group windows: 'search' = configs/<model>_windows_w8.json (8-bit windows at "
                        "the window search's per-group k, tools/search_resnet.py) when present, 'uniform' = (k, m) for every group, or a ReluConfig JSON path")
    p.add_argument("--no-model-graph", action="store_true",
                   help="ResNet: launch the forward's kernels one by one instead of replaying it as one CUDA graph")
    p.add_argument("--resnet-triple-gb", type=float, default=100.0,
                   help="HBM budget for one ResNet micro-batch's triples (both parties)")
    p.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                   help="N>1 exchange backend (gloo lets 2 ranks share one GPU for testing)")
    p.add_argument("--spawn-selftest", action="store_true",
                   help="CPU check of the --gpus N self-launch: ranks join a gloo group, rank 0 reports")
    return p.parse_args()


# ------------------------------------------------------------------ measured peaks / clocks
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Polls NVML (SM clock, throttle reasons) from a thread while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons, self.period = [], 0, period
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # noqa: BLE001
            log(f"[clocks] NVML unavailable: {exc}")
            self.nv = None
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ workload
def algorithmic_bytes_per_elem(w: int, ring_bits: int, levels: int) -> dict:
    """HBM bytes per element per party (DESIGN.md section 'roofline').

    fused:  x (8) + y (8) + bool triples 3(1+2L)w/8 + arith triples 2*3*N/8; the
            openings never leave the SM (shared-memory wire).
    survey: SURVEY.md 8(d) H(w) = fused + 2 W(w) (own openings written, peer's read)."""
    bool_b = 3 * (1 + 2 * levels) * w / 8
    arith_b = 6 * ring_bits / 8
    wire = (2 * w + 4 * levels * w) / 8 + 2 * 2 * ring_bits / 8
    fused = 16 + bool_b + arith_b
    return {"fused": fused, "survey_H": fused + 2 * wire, "wire_W": wire}


def device_inputs(n, ring_bits, seed, device):
    """x_f ~ N(0, 4^2) encoded at f = 16 and split (x + r, -r), generated in HBM."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    xf = torch.randn(n, generator=g, device=device, dtype=torch.float64) * 4.0
    e = (torch.sign(xf) * torch.floor(xf.abs() * 65536.0 + 0.5)).to(torch.int64)
    r = torch.bitwise_or(torch.bitwise_left_shift(torch.empty(n, dtype=torch.int64, device=device)
                                                  .random_(0, 1 << 32, generator=g), 32),
                         torch.empty(n, dtype=torch.int64, device=device).random_(0, 1 << 32, generator=g))
    if ring_bits < 64:
        e, r = e & ((1 << ring_bits) - 1), r & ((1 << ring_bits) - 1)
    x0, x1 = e + r, -r
    if ring_bits < 64:
        x0, x1 = x0 & ((1 << ring_bits) - 1), x1 & ((1 << ring_bits) - 1)
    return x0, x1


def stock_sets(stores, parties, n, w, ring_bits, levels, budget_gb, want_sets, seed):
    """Stock `sets` steps' worth of triples (fresh per step if they fit the HBM budget)."""
    from paper_2309_04875_b200 import dealer

    per_step = len(parties) * n * (3 * (1 + 2 * levels) * w / 8 + 6 * ring_bits / 8)
    sets = int(max(1, min(want_sets, budget_gb * 1e9 // max(per_step, 1))))
    nb, na = n * (1 + 2 * levels) * sets, 2 * n * sets
    dealer.stock_on_device(stores, parties, dealer.BOOL, w, nb, seed)
    dealer.stock_on_device(stores, parties, dealer.ARITH, ring_bits, na, seed + 1)
    return sets


def check_sample(x0, x1, y0, y1, ring_bits, k, m, count=1 << 20):
    """Reconstruction == x * drelu_from_shares on a sample (host check, not timed)."""
    from oracle import hb_oracle as O

    c = min(count, x0.numel())
    h = [t[:c].cpu().numpy().view(np.uint64) for t in (x0, x1, y0, y1)]
    want = O.ring_mul(O.ring_add(h[0], h[1], ring_bits), O.drelu_from_shares(h[0], h[1], ring_bits, k, m), ring_bits)
    return bool(np.array_equal(O.ring_add(h[2], h[3], ring_bits), want))


def cpu_baseline(k, m, ring_bits, steps=2, warmup=1):
    """The reference algorithm on the box's host cores (see ref_parallel)."""
    value, step_s, workers, eff = ref_parallel(k, m, ring_bits, steps, warmup)
    return {"value": value, "unit": UNIT, "cores": 2 * workers, "effective_cores": round(eff, 2),
            "host_cpu_count": os.cpu_count(), "kind": "port",
            "sample": f"{steps} steps of {workers} x 2^17-element chunks, window ({k},{m}); one reference-algorithm "
                      f"pair (oracle/hb_oracle.py incl. unpackbits codec, 2 party threads) per worker process"}


def model_baselines(cpu_relu_rate, batch=64):
    """SURVEY 8(d) model-level context on this host (untimed by the bench clock, N = 1 only):
    * desk_cnn: the reference's desk CNN (models.py:50-72; weights = the reference's own draws, the
      same generator) through run_local_forward (cli.py:159-180) -- the reference algorithm on the host
      (oracle port, 2 party threads) vs this package on the GPU (pair mode, numpy in / logits out),
      same inputs, seed and windows; the logits must be identical.
    * resnet18_cpu_estimate: seconds per sample for ONE party pair on the host, an ESTIMATE (the
      reference cannot express residual blocks): ReLU elements / the measured host ReLU rate (all
      cores) + 2 x conv MACs / the measured host ring-conv MAC rate (oracle conv2d, uint64 matmul,
      on a layer1-shaped conv of one image)."""
    import numpy as np

    from oracle import hb_oracle_nn as ON
    from paper_2309_04875_b200 import models, nn
    from paper_2309_04875_b200.ring import BitWindow

    model = models.desk_cnn(11)
    wins = [BitWindow(20, 8), BitWindow(19, 6)]
    cfg = nn.ReluConfig(wins)
    x_f = np.random.default_rng(2024).uniform(0.0, 1.0, (batch, 1, 8, 8))
    layers = [nn._layer_to_json(L) for L in model.layers]
    t0 = time.perf_counter()
    ref_logits, _, _ = ON.run_local_forward(layers, model.input_shape, model.weights, [(w.k, w.m) for w in wins],
                                            x_f, 5)
    t_cpu = time.perf_counter() - t0  # includes the host dealer (the reference's run_local_forward excludes it)
    nn.run_local_forward(model, cfg, x_f, 5, pair=True)  # warm-up (kernel loads, weight encoding)
    logits, _, _, gpu_ms = nn.run_local_forward(model, cfg, x_f, 5, pair=True)
    desk = {"batch": batch, "windows": [[w.k, w.m] for w in wins], "seed": 5,
            "cpu_samples_per_s": batch / t_cpu, "cpu_cores": 2, "cpu_kind": "port",
            "cpu_note": "oracle/hb_oracle_nn.run_local_forward (reference algorithm, 2 party threads); wall "
                        "includes the host dealer",
            "gpu_samples_per_s": batch / (gpu_ms / 1e3),
            "gpu_note": "nn.run_local_forward(pair=True) wall_ms (host shares in, logits out; dealer excluded, "
                        "as cli.py:170-177 times it)",
            "logits_identical": bool(np.array_equal(logits, ref_logits))}
    # ring-conv MAC rate of the reference algorithm on this host (one party, one image, layer1 shape)
    rng = np.random.default_rng(3)
    xs = rng.integers(0, 2**63, (1, 64, 32, 32), dtype=np.uint64)
    wt = rng.normal(0, 0.05, (64, 64, 3, 3)).astype(np.float32)
    t0 = time.perf_counter()
    ON.conv2d(xs, 0, 64, 64, 3, 3, 1, 1, wt, np.zeros(64, np.float32))
    conv_rate = 64 * 64 * 9 * 32 * 32 / (time.perf_counter() - t0)
    rn = models.resnet18_cifar(0)
    relu_per_sample = sum(c for _, c in rn.relu_sites())
    macs = models.conv_macs(rn)
    est = relu_per_sample / cpu_relu_rate + 2 * macs / conv_rate
    return desk, {"seconds_per_sample_per_pair": est, "label": "ESTIMATE (not a run)",
                  "relu_elems_per_sample": relu_per_sample, "host_relu_elems_per_s": cpu_relu_rate,
                  "conv_macs_per_sample": macs, "host_conv_macs_per_s_per_party": conv_rate,
                  "samples_per_s": 1.0 / est}


# ------------------------------------------------------------------ N = 1: fused pair
def run_single(args):
    import torch

    from paper_2309_04875_b200 import dealer, protocol, transport
    from paper_2309_04875_b200.protocol import ProtocolSession
    from paper_2309_04875_b200.ring import BitWindow
    from paper_2309_04875_b200.sharing import ArithShareTensor

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    from paper_2309_04875_b200 import _dev as _hb_dev

    _hb_dev.bind_thread()  # the library's own CUDA runtime on this rank's device
    n, k, m, N = 1 << args.logn, args.k, args.m, args.ring_bits
    w = k - m
    L = protocol.prefix_levels(w)
    win = BitWindow(k, m)
    eps = transport.local_pair()
    stores = (dealer.TripleStore(0), dealer.TripleStore(1))
    sessions = (ProtocolSession(eps[0], stores[0]), ProtocolSession(eps[1], stores[1]))
    x0, x1 = device_inputs(n, N, 1234, dev)
    sets = stock_sets(stores, (0, 1), n, w, N, L, args.triple_gb, args.steps + args.warmup, seed=99)
    need = {(dealer.BOOL, w): n * (1 + 2 * L), (dealer.ARITH, N): 2 * n}
    s = torch.cuda.current_stream()
    if args.path == "p2p":
        links = transport.local_p2p_pair()

    def step(a0, a1):
        if stores[0].remaining(dealer.BOOL, w) < need[(dealer.BOOL, w)]:
            for st in stores:
                st.rewind(dealer.BOOL, w)
                st.rewind(dealer.ARITH, N)
        if args.path == "pair":
            return protocol.relu_pair(sessions, ArithShareTensor(0, N, a0), ArithShareTensor(1, N, a1), win)
        if args.path == "p2p":  # both party kernels in one launch on this device, openings via peer buffers
            return protocol.relu_p2p_pair(sessions, ArithShareTensor(0, N, a0), ArithShareTensor(1, N, a1), win, links,
                                          sys_scope=args.p2p_scope == "sys")
        return transport.run_parties(lambda: protocol.relu(sessions[0], ArithShareTensor(0, N, a0), win),
                                     lambda: protocol.relu(sessions[1], ArithShareTensor(1, N, a1), win))

    for _ in range(args.warmup):
        y0, y1 = step(x0, x1)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    graph = None
    if args.graph:  # the timed steps as one CUDA graph: what the GPU sustains without host launch gaps
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(args.steps):
                y0, y1 = step(x0, x1)
        graph.replay()  # warm
        torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t_start.record(s)
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                ev[i][0].record(s)
                y0, y1 = step(x0, x1)
                ev[i][1].record(s)
        t_end.record(s)
        torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    launch_ms = (total_ms / args.steps if graph is not None
                 else statistics.mean(a.elapsed_time(b) for a, b in ev))
    ok = check_sample(x0, x1, y0.data, y1.data, N, k, m)
    value = n * args.steps / (total_ms / 1e3)

    bpe = algorithmic_bytes_per_elem(w, N, L)
    peak, peak_src = peaks()
    # the P2P kernels write the openings to the peer's buffer and read the peer's: SURVEY H(w)
    alg_bpe = bpe["survey_H"] if args.path == "p2p" else bpe["fused"]
    alg_bytes = 2 * n * alg_bpe
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    # the timed kernel's instantiation (as ncu prints it) and its committed --set full capture, used
    # only when the capture is of this very kernel at this size
    if args.path == "p2p":
        kernel = f"k_relu_p2p<{w}>"
        key = f"p2p_{args.p2p_scope}_w{w}_n{args.logn}"
    else:
        kernel = f"k_relu_pair<{w}, 32, {1 if N == 64 else 0}>"
        key = f"pair_w{w}_n{args.logn}"
    traffic = traffic_src = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            prof = json.load(fh)
        if key in prof and kernel in prof[key]["kernel"]:
            traffic = prof[key]["dram_bytes_per_launch"]
            traffic_src = f"profiles/ncu_summary.json[{key}] ({prof[key]['kernel']})"
    except (OSError, ValueError, KeyError):
        pass

    if args.path == "p2p":
        for lk in links:
            lk.check(sync=True)
    # ---- e2e: the public API with host (pinned) buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e and args.path == "pair":
        # both parties' input shares in one pinned [2, n] staging buffer (one two-row H2D per chunk)
        hb = torch.stack([x0, x1]).cpu().pin_memory()
        h0, h1 = hb[0], hb[1]
        torch.cuda.synchronize()
        reps = max(3, min(args.steps, 10))
        for _ in range(3):  # populate the pinned-buffer cache the way the timed loop uses it
            r0, r1 = step(h0, h1)
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r0, r1 = step(h0, h1)
            _ = (r0.data, r1.data)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        log(f"[e2e] per-step ms: {[round(1e3 * t, 2) for t in times]}")
        dt = sum(times)
        e2e = {"value": n * reps / dt, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * n, "d2h_bytes_per_step": 2 * 8 * n,
               "path": "protocol.relu_pair with pinned host shares in (one [2, n] staging buffer) and host shares out", "steps": reps}

    cpu = None if args.no_cpu_baseline else cpu_baseline(k, m, N)
    desk = rn_est = None
    if cpu is not None and args.path == "pair":
        desk, rn_est = model_baselines(cpu["value"])
    resnet = None
    if not args.no_resnet and args.path == "pair" and args.logn == 24:
        del stores, sessions, x0, x1, y0, y1
        torch.cuda.empty_cache()
        import copy

        ra = copy.copy(args)
        ra.workload, ra.batch, ra.steps, ra.warmup = "resnet18", 512, 3, 2
        r = run_resnet(ra)
        resnet = {"metric": r["metric"], "value": r["value"], "unit": r["unit"], "ms_per_step": r["ms_per_step"],
                  "config": r["config"], "steps": r["steps"], "warmup": r["warmup"],
                  "logits_check": r["logits_check"], "cpu_estimate": rn_est,
                  "layer_breakdown": r["layer_breakdown"]}
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"secure ReLU layer n=2^{args.logn}, window ({k},{m}) w={w}, N={N}",
                   "n": n, "window": [k, m], "ring_bits": N, "parties": "1 pair time-sliced on 1 GPU",
                   "path": {"pair": "fused pair kernel hb_relu_pair", "staged": "staged hb_relu_round x2",
                            "p2p": "both parties' NVLink party kernels in one launch (hb_relu_p2p_pair), openings via "
                                   f"each other's receive buffers, {args.p2p_scope}-scope flags"}[args.path],
                   "inputs": "x_f~N(0,4^2), f=16, additive shares; Beaver triples from the on-device dealer",
                   "triple_sets": sets, "l2": f"inputs {2 * n * bpe['fused'] / 1e9:.2f} GB/step > 126 MB L2",
                   "cuda_graph": bool(args.graph),
                   "parallelism": "pair"},
        "correct": ok,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_elem_per_party": alg_bpe, "survey_H_bytes_per_elem_per_party": bpe["survey_H"],
                     "frac_vs_survey_H": (2 * n * bpe["survey_H"] / (launch_ms / 1e3) / 1e9) / peak,
                     "kernel": "hb::" + kernel, "traffic_source": traffic_src, "launch_ms": launch_ms,
                     "peak_note": "peak = the driver's copy benchmark (1 read : 1 write); the ReLU kernels mostly "
                                  "read (x and the triples; w = 8: 77 of 85 B per element and party) and read-only "
                                  "streaming reaches ~6.83 TB/s on these boxes (profiles/hbm_stream_rates_r02.json), "
                                  "so frac can exceed 1"},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps, "clocks": clk.summary(),
        "resnet18": resnet, "desk_cnn": desk,
    }


# ------------------------------------------------------------------ ResNet private inference (N = 1)
def resnet_windows(args, model):
    """(ReluConfig, description) for a ResNet run: the committed window-search result by default
    (BASELINE configs[2]: per-layer (k, m) from the search config), else one window for all groups."""
    from paper_2309_04875_b200 import models, nn
    from paper_2309_04875_b200.ring import BitWindow

    path = args.relu_config
    if path == "search":
        path = os.path.join(ROOT, "configs", f"{args.workload}_windows_w8.json")
        if not os.path.exists(path):
            path = "uniform"
    if path == "uniform":
        return models.resnet_relu_config(model, BitWindow(args.k, args.m)), f"all groups ({args.k},{args.m})"
    with open(path) as fh:
        obj = json.load(fh)
    cfg = nn.ReluConfig.from_json(obj)
    if len(cfg.windows) != model.n_groups:
        raise SystemExit(f"{path}: {len(cfg.windows)} windows for {model.n_groups} groups")
    wins = ",".join("id" if w is None else f"({w.k},{w.m})" for w in cfg.windows)
    return cfg, f"per group {wins} from {os.path.relpath(path, ROOT)}"


def micro_batch(model, cfg, batch, parties, budget_gb):
    """Largest power-of-two split of `batch` whose (a, b, c) triple streams for `parties` parties fit
    `budget_gb` of HBM (the batch's triples are read once per forward; they are not reusable)."""
    from paper_2309_04875_b200 import nn

    def triple_bytes(b):
        return sum(3 * parties * (-(-c * w // 64) * 8 if kind == "bool" else 8 * c)
                   for (kind, w), c in nn.triple_requirements(model, cfg, b).items())

    mb = batch
    while mb > 1 and triple_bytes(mb) > budget_gb * 2**30:
        mb //= 2
    if batch % mb:
        raise SystemExit(f"batch {batch} does not split into micro-batches of {mb}")
    return mb


def run_resnet(args):
    """ResNet private inference samples/s, both parties time-sliced on one GPU (BASELINE configs[2,3])."""
    import torch

    from paper_2309_04875_b200 import dealer, models, nn, transport
    from paper_2309_04875_b200.protocol import ProtocolSession
    from paper_2309_04875_b200.ring import BitWindow
    from paper_2309_04875_b200.sharing import ArithShareTensor

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    from paper_2309_04875_b200 import _dev as _hb_dev

    _hb_dev.bind_thread()  # the library's own CUDA runtime on this rank's device
    if args.workload == "resnet18":
        model, batch, shape = models.resnet18_cifar(0), args.batch or 512, (3, 32, 32)
    else:
        model, batch, shape = models.resnet50(0), args.batch or 128, (3, 64, 64)
    cfg, cfg_desc = resnet_windows(args, model)

    # micro-batches when the whole batch's triples exceed the HBM budget (ResNet50 b128 at 64x64
    # needs ~208 GB); each micro-batch forward reads its full triple stock from HBM, and the stock
    # is rewound between micro-batches and steps (the dealer is the offline phase, not timed)
    mb = micro_batch(model, cfg, batch, 2, args.resnet_triple_gb)
    need = nn.triple_requirements(model, cfg, mb)
    eps = transport.local_pair()
    stores = (dealer.TripleStore(0), dealer.TripleStore(1))
    for i, ((kind, width), count) in enumerate(sorted(need.items())):
        dealer.stock_on_device(stores, (0, 1), kind, width, count, seed=500 + i)
    sessions = (ProtocolSession(eps[0], stores[0], model.fixed_point), ProtocolSession(eps[1], stores[1], model.fixed_point))
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    x_f = torch.rand((batch,) + shape, generator=g, device=dev, dtype=torch.float64)
    enc = torch.floor(x_f * 65536.0 + 0.5).to(torch.int64)
    r = torch.empty_like(enc).random_(generator=g)
    x0s = [ArithShareTensor(0, 64, (enc + r)[i:i + mb]) for i in range(0, batch, mb)]
    x1s = [ArithShareTensor(1, 64, (-r)[i:i + mb]) for i in range(0, batch, mb)]
    s = torch.cuda.current_stream()

    def fwd():
        out = None
        for x0, x1 in zip(x0s, x1s):
            for st in stores:
                for (kind, width) in need:
                    st.rewind(kind, width)
            out = nn.model_forward_pair(sessions, x0, x1, model, cfg)
        return out

    for _ in range(args.warmup):
        y0, y1 = fwd()
    torch.cuda.synchronize()
    graph = None
    if not args.no_model_graph:
        # the whole forward (every micro-batch, both parties: ~110 kernels) as ONE CUDA graph: the same
        # kernels on the same buffers, without the host's per-launch gaps between them
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            y0, y1 = fwd()
        graph.replay()
        torch.cuda.synchronize()

    def step():
        if graph is not None:
            graph.replay()
            return y0, y1
        return fwd()

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(args.steps):
            y0, y1 = step()
        b.record(s)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    relu_elems = sum(c for _, c in model.relu_sites()) * batch
    # sampled fidelity check (untimed): the reconstructed logits of the last micro-batch's first 8
    # images against the exact float forward of the same inputs (simulator.plain_forward)
    from paper_2309_04875_b200 import simulator

    k8 = min(8, mb)
    rec = (y0.data[:k8] + y1.data[:k8]).cpu().numpy().astype(np.int64).astype(np.float64) / 65536.0
    plain = simulator.plain_forward(model, x_f[batch - mb:batch - mb + k8].cpu().numpy())
    logits_check = {"images": k8, "max_abs_diff_vs_plain_forward": float(np.max(np.abs(rec - plain))),
                    "argmax_agree": int(np.sum(np.argmax(rec, 1) == np.argmax(plain, 1))),
                    "plain_logit_absmax": float(np.max(np.abs(plain)))}
    # per-layer device time of one (untimed, un-captured) micro-batch forward from CUDA events
    # (nn.model_forward_pair(layer_times=...)), summed by layer kind; a residual block's own time is
    # its fused last conv (+ the residual add) -- its entry minus its direct children's
    for _ in range(2):  # the first eager pass populates the caching allocator outside the graph's pool
        times = []
        for st in stores:
            for (kind, width) in need:
                st.rewind(kind, width)
        nn.model_forward_pair(sessions, x0s[0], x1s[0], model, cfg, layer_times=times)
    by_kind = {}
    for t in times:
        ms_self = t["ms"]
        if t["kind"] == "residual":
            depth = t["layer"].count(".")
            ms_self -= sum(u["ms"] for u in times if u["layer"].startswith(t["layer"] + ".")
                           and u["layer"].count(".") == depth + 2)
        key = "conv2d" if t["kind"] == "residual" else t["kind"]
        by_kind[key] = by_kind.get(key, 0.0) + ms_self
    layer_breakdown = {"micro_batch": mb, "ms_by_kind": {k: round(v, 3) for k, v in by_kind.items()},
                       "note": "second eager forward (no CUDA graph), CUDA events per layer (host launch gaps "
                               "included); conv2d includes the limb-plane split and the fused residual add"}
    return {
        "metric": f"{args.workload}_private_inference_samples_per_s", "value": batch / (ms / 1e3),
        "unit": "samples/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{args.workload} private inference, batch {batch}, input {shape}, "
                               f"ReLU windows {cfg_desc}", "batch": batch,
                   "relu_elements_per_forward": relu_elems, "parties": "1 pair time-sliced on 1 GPU",
                   "micro_batch": mb, "stem": "CIFAR-style 3x3 stride 1, no maxpool",
                   "cuda_graph": graph is not None,
                   "path": "nn.model_forward_pair: int8-limb ring conv ("
                           + ("hand-written tcgen05 kernel" if nn.RING_GEMM == "tc" else "cuBLASLt") + ") + fused pair ReLU kernel",
                   "weights": "random init (torchvision scheme), BN folded", "parallelism": "pair"},
        "relu_elems_per_s_in_model": relu_elems / (ms / 1e3), "logits_check": logits_check, "clocks": clk.summary(),
        "layer_breakdown": layer_breakdown,
    }


# ------------------------------------------------------------------ N > 1: party pairs over NCCL
def run_multi(args):
    import torch
    import torch.distributed as dist

    from paper_2309_04875_b200 import dealer, protocol, transport
    from paper_2309_04875_b200.protocol import ProtocolSession
    from paper_2309_04875_b200.ring import BitWindow
    from paper_2309_04875_b200.sharing import ArithShareTensor

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2309_04875_b200 import _dev as _hb_dev

    _hb_dev.bind_thread()  # the library's own CUDA runtime on this rank's device
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
        args.triple_gb = min(args.triple_gb, 16.0)
    pairs = world // 2
    pair, party = rank // 2, rank % 2
    active = pair < pairs
    if args.workload != "relu":
        return run_multi_resnet(args, dist, dev, rank, world, pairs, pair, party, active)
    n, k, m, N = 1 << args.logn, args.k, args.m, args.ring_bits
    w = k - m
    L = protocol.prefix_levels(w)
    win = BitWindow(k, m)
    ep = transport.DistEndpoint(party, rank ^ 1) if active else None
    if active and args.multi_path == "p2p" and ep.enable_p2p() is None:
        log(f"[rank {rank}] NVLink P2P mapping unavailable: staged rounds + {args.backend}")
    used_p2p = bool(active and ep.p2p is not None)
    store = dealer.TripleStore(party)
    s = torch.cuda.current_stream()
    if active:
        # both ranks of a pair derive the same dealt values from the pair seed and keep their own share
        x0, x1 = device_inputs(n, N, 1234 + pair, dev)
        mine = (x0, x1)[party]
        del x0, x1
        sets = stock_sets((store,), (party,), n, w, N, L, args.triple_gb, args.steps + args.warmup, seed=99 + 7 * pair)
        sess = ProtocolSession(ep, store)
    need_b = n * (1 + 2 * L)

    def step():
        if store.remaining(dealer.BOOL, w) < need_b:
            store.rewind(dealer.BOOL, w)
            store.rewind(dealer.ARITH, N)
        return protocol.relu(sess, ArithShareTensor(party, N, mine), win)

    y = None
    if active:
        for _ in range(args.warmup):
            y = step()
    torch.cuda.synchronize()
    dist.barrier()
    graph = None
    if args.graph and used_p2p:
        # each party rank's timed steps as ONE CUDA graph: the party kernel's flag sequence and receive
        # region live on the device (PeerLink.state), so the replays of the two ranks stay in step
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(args.steps):
                y = step()
        graph.replay()  # warm (the partner rank replays too)
        torch.cuda.synchronize()
        ep.p2p.check(sync=True)
        dist.barrier()
    with ClockSampler(local) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        a.record(s)
        if graph is not None:
            graph.replay()
        elif active:
            for _ in range(args.steps):
                y = step()
        b.record(s)
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([a.elapsed_time(b)], device=dev if args.backend == "nccl" else "cpu")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    # correctness (untimed): partners swap a sample of x / y shares, party 0 reconstructs
    ok = torch.ones(1, device=ms.device)
    if active:
        c = min(n, 1 << 20)
        mine_s = torch.cat([mine[:c], y.data.reshape(-1)[:c]])
        theirs = ep._swap(mine_s)
        if not isinstance(theirs, torch.Tensor):
            theirs = torch.from_numpy(np.frombuffer(theirs, dtype=np.int64).copy())
        theirs = theirs.to(dev)
        if party == 0:
            ok[0] = float(check_sample(mine_s[:c], theirs[:c], mine_s[c:], theirs[c:], N, k, m))
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # e2e: the public per-party call with this rank's share in pinned host memory -- H2D of the share,
    # the ReLU, D2H of the output share inside the timed region -- max over ranks
    e2e = None
    if not args.no_e2e:
        h_in = mine.cpu().pin_memory() if active else None
        h_out = torch.empty(n, dtype=torch.int64, pin_memory=True) if active else None
        reps = max(3, min(args.steps, 10))

        def e2e_step():
            xd = h_in.to(dev, non_blocking=True)
            yv = step_on(xd)
            h_out.copy_(yv.data.reshape(-1), non_blocking=True)

        def step_on(xd):
            if store.remaining(dealer.BOOL, w) < need_b:
                store.rewind(dealer.BOOL, w)
                store.rewind(dealer.ARITH, N)
            return protocol.relu(sess, ArithShareTensor(party, N, xd), win)

        if active:
            e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        if active:
            for _ in range(reps):
                e2e_step()
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], device=ms.device)
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e = {"value": pairs * n * reps / float(el.item()), "unit": UNIT, "h2d_bytes_per_step": world * 8 * n,
               "d2h_bytes_per_step": world * 8 * n, "steps": reps,
               "path": "protocol.relu per party rank with its share in pinned host memory in and out (max over ranks)"}
    out = None
    if rank == 0:
        value = pairs * n * args.steps / (total_ms / 1e3)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"secure ReLU layer n=2^{args.logn} per pair, window ({k},{m}) w={w}, N={N}",
                       "n_per_pair": n, "pairs": pairs, "window": [k, m], "ring_bits": N,
                       "path": ("one-launch NVLink party kernel hb_relu_p2p, openings stored into the peer's "
                                "buffer (CUDA IPC) with per-chunk flags (ranks 2i<->2i+1)") if used_p2p
                       else f"staged hb_relu_round + {args.backend} send/recv per round (ranks 2i<->2i+1)",
                       "cuda_graph": graph is not None, "parallelism": f"{pairs} party pairs"},
            "gpu_launches": args.steps * (1 if used_p2p else L + 4), "clocks": clk.summary(),
            "correct": bool(ok.item() > 0.5),
            "e2e": e2e,
        }
    dist.destroy_process_group()
    return out


def run_multi_resnet(args, dist, dev, rank, world, pairs, pair, party, active):
    """ResNet private inference on `pairs` party pairs (ranks 2i/2i+1), batch sharded over pairs
    (BASELINE configs[4]: ResNet18 batch 4096 on 4 pairs).  Each rank runs nn.model_forward for
    its party; every ReLU round is a send/recv with its partner rank."""
    import torch

    from paper_2309_04875_b200 import dealer, models, nn, transport
    from paper_2309_04875_b200.protocol import ProtocolSession
    from paper_2309_04875_b200.ring import BitWindow
    from paper_2309_04875_b200.sharing import ArithShareTensor

    if args.workload == "resnet18":
        model, total, shape = models.resnet18_cifar(0), args.batch or 4096, (3, 32, 32)
    else:
        model, total, shape = models.resnet50(0), args.batch or 512, (3, 64, 64)
    per_pair = max(1, total // max(pairs, 1))
    cfg, cfg_desc = resnet_windows(args, model)
    # one party per rank: its own triple streams only, micro-batched to the HBM budget (configs[4] at
    # 2 GPUs is one pair x 4096 samples = ~155 GB of triples per party)
    mb = micro_batch(model, cfg, per_pair, 1, args.resnet_triple_gb)
    s = torch.cuda.current_stream()
    used_p2p = False
    if active:
        ep = transport.DistEndpoint(party, rank ^ 1)
        if args.multi_path == "p2p" and ep.enable_p2p() is None:
            log(f"[rank {rank}] NVLink P2P mapping unavailable: staged rounds + {args.backend}")
        used_p2p = ep.p2p is not None
        store = dealer.TripleStore(party)
        need = nn.triple_requirements(model, cfg, mb)
        for i, ((kind, width), count) in enumerate(sorted(need.items())):
            dealer.stock_on_device((store,), (party,), kind, width, count, seed=500 + 31 * pair + i)
        sess = ProtocolSession(ep, store, model.fixed_point)
        g = torch.Generator(device=dev)
        g.manual_seed(7 + pair)  # both ranks of a pair derive the same split, keep their own share
        x_f = torch.rand((per_pair,) + shape, generator=g, device=dev, dtype=torch.float64)
        enc = torch.floor(x_f * 65536.0 + 0.5).to(torch.int64)
        r = torch.empty_like(enc).random_(generator=g)
        share = enc + r if party == 0 else -r
        mines = [ArithShareTensor(party, 64, share[i:i + mb]) for i in range(0, per_pair, mb)]
        x_check = x_f[per_pair - mb:per_pair - mb + min(8, mb)].cpu().numpy()  # the last micro-batch's first images
        del x_f, enc, r

    def fwd():
        out = None
        for mine in mines:
            for (kind, width) in need:
                store.rewind(kind, width)
            out = nn.model_forward(sess, mine, model, cfg)
        return out

    if active:
        for _ in range(args.warmup):
            fwd()
    torch.cuda.synchronize()
    dist.barrier()
    with ClockSampler(dev.index) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        a.record(s)
        if active:
            for _ in range(args.steps):
                fwd()
        b.record(s)
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([a.elapsed_time(b)], device=dev if args.backend == "nccl" else "cpu")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    # fidelity (untimed): partners swap the logits shares of the last micro-batch's first images,
    # party 0 reconstructs them and compares with the exact float forward of the same inputs
    err = torch.zeros(1, device=ms.device)
    if active:
        last = fwd()
        k8 = x_check.shape[0]
        mine_l = last.data[:k8].reshape(-1).contiguous()
        theirs = ep._swap(mine_l)
        if not isinstance(theirs, torch.Tensor):
            theirs = torch.from_numpy(np.frombuffer(theirs, dtype=np.int64).copy())
        if party == 0:
            from paper_2309_04875_b200 import simulator

            rec = (mine_l.cpu() + theirs.cpu().reshape(-1)).numpy().astype(np.float64) / 65536.0
            plain = simulator.plain_forward(model, x_check).reshape(-1)
            err[0] = float(np.max(np.abs(rec - plain)))
    dist.all_reduce(err, op=dist.ReduceOp.MAX)
    out = None
    if rank == 0:
        out = {
            "logits_check": {"images_per_pair": int(x_check.shape[0]) if active else 0,
                             "max_abs_diff_vs_plain_forward": float(err.item())},
            "metric": f"{args.workload}_private_inference_samples_per_s",
            "value": pairs * per_pair * args.steps / (total_ms / 1e3), "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"{args.workload} private inference, batch {pairs * per_pair} over {pairs} pairs, "
                                   f"ReLU windows {cfg_desc}",
                       "batch": pairs * per_pair, "batch_per_pair": per_pair, "pairs": pairs, "micro_batch": mb,
                       "path": "nn.model_forward per party, ReLU " + (
                           "one-launch NVLink party kernel (openings into the peer's buffer)" if used_p2p
                           else f"staged + {args.backend} send/recv per round"),
                       "parallelism": f"{pairs} party pairs"},
            "clocks": clk.summary(), "e2e": None,
        }
    dist.destroy_process_group()
    return out


# ------------------------------------------------------------------ reference arm
_REF_BARRIER = None


def _ref_init(barrier):
    global _REF_BARRIER
    _REF_BARRIER = barrier


def _ref_task(job):
    """Worker: build one chunk's shares and dealt triples (not timed), wait for every worker,
    then run one reference-algorithm ReLU (two party threads) on it (timed)."""
    from oracle import hb_oracle as O

    idx, n, k, m, N, step = job
    rng = np.random.default_rng([2024, idx])
    x0, x1 = O.split_additive(O.encode_fixed(rng.normal(0, 4, n), 16, N), N, rng)
    curs = O.stocked_cursors(n, k - m, N, seed=1000 * step + idx)
    _REF_BARRIER.wait()
    t0, c0 = time.perf_counter(), time.process_time()
    O.relu_pair(x0, x1, N, k, m, curs)
    return t0, time.perf_counter(), time.process_time() - c0


def ref_parallel(k, m, N, steps, warmup, chunk=1 << 17):
    """Time the reference algorithm on all host cores: one pair (2 party threads) per two cores,
    each worker on its own chunk.  Returns (elements/s, wall s per step, workers, effective cores)."""
    import multiprocessing as mp

    workers = max(1, (os.cpu_count() or 2) // 2)
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(workers)
    walls, cpus = [], []
    with ctx.Pool(workers, initializer=_ref_init, initargs=(barrier,)) as pool:
        for i in range(warmup + steps):
            # one task per worker: each blocks at the barrier, so no worker takes two
            res = pool.map(_ref_task, [(w, chunk, k, m, N, i) for w in range(workers)], chunksize=1)
            # CLOCK_MONOTONIC is system-wide: the step spans first start to last finish
            wall = max(r[1] for r in res) - min(r[0] for r in res)
            if i >= warmup:
                walls.append(wall)
                cpus.append(sum(r[2] for r in res))
    wall = sum(walls)
    return workers * chunk * len(walls) / wall, wall / len(walls), workers, sum(cpus) / wall


def run_reference(args):
    """The reference algorithm (oracle port of ringmpc protocol.relu, two party threads per
    pair, byte-per-bit codec) on the host: one pair per two cores, each on its own chunk."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return None
    k, m, N = args.k, args.m, args.ring_bits
    value, step_s, workers, eff = ref_parallel(k, m, N, args.steps, args.warmup)
    sample = (f"per step {workers} x 2^17-element chunks of the 2^{args.logn} ReLU layer, window ({k},{m}), one "
              f"reference-algorithm pair (oracle/hb_oracle.py, 2 party threads) per worker process; "
              f"share/triple generation excluded")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"secure ReLU layer n=2^{args.logn}, window ({k},{m}) w={k - m}, N={N}",
                   "n": 1 << args.logn, "window": [k, m], "ring_bits": N, "parallelism": f"host, {workers} processes"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 2 * workers, "kind": "port", "sample": sample,
                         "effective_cores": round(eff, 2), "host_cpu_count": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------------ sweep
def run_sweep(args):
    import copy

    rows = []
    for logn in (16, 18, 20, 22, 24, 26):
        for k, m in ((64, 0), (32, 0), (22, 6), (22, 14), (22, 16)):
            a = copy.copy(args)
            a.logn, a.k, a.m = logn, k, m
            a.no_e2e, a.no_cpu_baseline, a.no_resnet = True, True, True
            # small layers: launch gaps would dominate the GPU time (the P2P path replays too: its flag
            # sequence and receive-region parity live on the device, advanced by the kernel itself)
            a.graph = logn <= 22 and args.path in ("pair", "p2p")
            a.steps = max(5, min(args.steps, 20))
            a.warmup = 3
            r = run_single(a)
            row = {"logn": logn, "k": k, "m": m, "w": k - m, "cuda_graph": a.graph, "elems_per_s": r["value"],
                   "ms_per_step": r["ms_per_step"], "hbm_frac": r["roofline"]["frac"],
                   "frac_vs_survey_H": r["roofline"]["frac_vs_survey_H"], "correct": r["correct"]}
            log(json.dumps(row))
            rows.append(row)
            import gc

            import torch

            gc.collect()  # the P2P links of a same-process pair reference each other (device buffers)
            torch.cuda.empty_cache()
    with open(args.sweep, "w") as fh:
        json.dump(rows, fh, indent=1)


def spawn_cmd(argv, nproc, port):
    """The driver's own multi-GPU launch line: one rank per GPU, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def self_launch(args, argv):
    """`bench.py --gpus N` run without torchrun: re-launch as N ranks (one party per GPU; ranks 2i / 2i+1
    are the parties of pair i) and pass rank 0's JSON line through.  NCCL_DEBUG=INFO (INIT subsystem)
    puts the communicator lines -- one per rank and device -- on stderr."""
    import socket
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    if args.backend == "nccl":
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = spawn_cmd(argv, args.gpus, port)
    log(f"[bench] self-launch: {' '.join(cmd)}")
    return subprocess.run(cmd, env=env).returncode


def spawn_selftest(args):
    """--spawn-selftest: the self-launch plumbing on CPU (gloo): every rank joins, rank 0 reports."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    t = torch.tensor([rank + 1])
    dist.all_reduce(t)
    out = {"selftest": "spawn", "n_gpus": world, "rank_sum": int(t.item()), "pairs": world // 2,
           "party_of_rank": [r % 2 for r in range(world)], "pair_of_rank": [r // 2 for r in range(world)]}
    dist.destroy_process_group()
    return out if rank == 0 else None


def main():
    args = parse()
    if (args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference" and not args.sweep):
        sys.exit(self_launch(args, sys.argv[1:]))
    if args.spawn_selftest:
        out = spawn_selftest(args)
    elif args.impl == "reference":
        out = run_reference(args)
    elif args.sweep:
        run_sweep(args)
        return
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1:
        out = run_multi(args)
    elif args.workload != "relu":
        out = run_resnet(args)
    else:
        out = run_single(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
