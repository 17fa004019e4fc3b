"""Benchmark: SSNet secure inference of ResNet-152 at 224x224 (5 parties, t=2, verification on)
on B200, all parties co-resident per GPU, images sharded data-parallel across GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--workload resnet152-5pc]
    python bench.py --impl reference ...     # CPU oracle port of the reference path

One step = one secure inference of a batch of B synthetic images per GPU: input sharing,
the device trusted source (all masks), and the full online protocol (156 share GEMMs,
reshares, masked truncations / ReLUs / pools, residual adds, output reconstruction with
Reed-Solomon verification).  Prints ONE JSON line (rank 0).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (builder, k, n, verify, default batch per GPU)
    "resnet152-5pc": ("imagenet152", 3, 5, True, 64),
    "resnet152-3pc": ("imagenet152", 2, 3, True, 64),
    "resnet50-3pc": ("imagenet50", 2, 3, False, 64),
    "resnet18-cifar-3pc": ("cifar18", 2, 3, False, 256),
    "lenet-3pc": ("reference", 2, 3, False, 16384),
    "lenet28-3pc": ("lenet28", 2, 3, False, 8192),     # config 1: LeNet-style CNN on 1x28x28
    "gemm-sweep": ("gemm", 0, 0, False, 0),          # config 5: mod-p share GEMM + reshare sweep
}
SWEEP = [(256, 256, 256), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192),
         (16384, 4096, 4096), (4096, 4096, 16384), (16384, 16384, 16384)]
# default CUDA streams per GPU (co-resident placement).  S streams split the batch so one part's
# tensor-bound GEMMs overlap another's ALU-bound protocol chains (profiles/r01/README.md,
# batch/stream sweep).  The first timed step runs the sub-batches back to back: its per-kernel
# CUDA events give each kernel's own time for the rooflines; the remaining steps overlap.
DEFAULT_STREAMS = {"resnet152-5pc": 2, "resnet152-3pc": 2, "resnet50-3pc": 2, "resnet18-cifar-3pc": 2}
METRIC = "ResNet-152 secure-inference images/s (5PC t=2, verification on, 224x224)"


def build_model(kind):
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.model import build_reference_model
    if kind == "imagenet152":
        return resnet.imagenet_resnet(152)
    if kind == "imagenet50":
        return resnet.imagenet_resnet(50)
    if kind == "cifar18":
        return resnet.cifar_resnet18()
    if kind == "lenet28":
        from paper_2406_02629_b200.model import build_lenet28
        return build_lenet28(7, pool="max")[0]
    return build_reference_model(7, pool="max")[0]


def metric_for(workload):
    if workload == "resnet152-5pc":
        return METRIC
    if workload == "resnet152-3pc":
        return "ResNet-152 secure-inference images/s (3PC t=1, verification on, 224x224)"
    return f"{workload} secure-inference images/s"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML polled
    every 20 ms from a thread (so even a sub-second timed region gets samples), nvidia-smi as
    the fallback.  The last sample is always taken at stop()."""

    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.stop_evt = threading.Event()
        self.nv = None
        self.thread = None

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.samples.append((sm, mx, {nm for nm, attr in self.NAMES.items() if mask & getattr(nv, attr, 0)}))

    def _loop(self):
        while not self.stop_evt.wait(0.02):
            try:
                self._sample()
            except Exception:
                return

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self._sample()
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
        except Exception:
            self.nv = None

    def stop(self):
        if self.nv is None:
            return self._smi_once()
        self.stop_evt.set()
        self.thread.join(timeout=2)
        try:
            self._sample()
        except Exception:
            pass
        sms = [x[0] for x in self.samples]
        reasons = sorted(set().union(*[x[2] for x in self.samples])) if self.samples else []
        return {"sm_mhz": float(np.median(sms)) if sms else None,
                "sm_max_mhz": float(max(x[1] for x in self.samples)) if self.samples else None,
                "reasons": reasons, "samples": len(sms), "source": "nvml, 20 ms polling"}

    def _smi_once(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
            parts = [x.strip() for x in out.strip().split(",")]
            reasons = [nm for nm, v in zip(self.NAMES, parts[2:6]) if v.lower() == "active"]
            return {"sm_mhz": float(parts[0]), "sm_max_mhz": float(parts[1]), "reasons": reasons, "samples": 1,
                    "source": "nvidia-smi at stop (NVML unavailable)"}
        except Exception as exc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"clock query failed: {exc!r}"], "samples": 0}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("hbm_gbs", 6545.3), d.get("bf16_tflops_sustained", d.get("bf16_tflops", 1653.7)), "measured sustained"
    except OSError:
        return 6650.0, 1590.0, "fallback"


def measured_int8():
    """Dense int8 tensor-pipe TOP/s measured on a B200 with tools/int8_peak.py (ssn_mma_peak:
    back-to-back tcgen05.mma.kind::i8), committed as profiles/r*/int8_peak.json; None if absent."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "int8_peak.json")))
    if not files:
        return None
    try:
        with open(files[-1]) as fh:
            d = json.load(fh)
        return {"burst": float(d["int8_tops_burst"]), "sustained": float(d["int8_tops_sustained"]),
                "src": os.path.relpath(files[-1], ROOT)}
    except (OSError, KeyError, ValueError):
        return None


def burst_bf16():
    """Burst dense bf16 TF/s (best of 10, MEASURED_PEAKS.json); a short step's GEMMs can exceed
    the 4-second sustained figure, so the GEMM roofline states both fractions."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return 1590.0


def cpu_baseline_sample(model, k, n, verify, budget_s=20.0):
    """Time the CPU oracle port (oracle/sim.py lockstep protocol with the C arithmetic, all
    host threads) on a prefix of the same schedule for ONE image; extrapolate to the full
    network by field-MAC share (the oracle spends >95% in the share GEMM)."""
    import oracle
    from oracle import sim
    from paper_2406_02629_b200.layers import ScheduledOp, _flag_passive
    oracle.build()
    cores = oracle.set_threads(0)            # all host cores (torchrun exports OMP_NUM_THREADS=1)
    if not hasattr(model, "nodes"):          # chain models (ModelGraph): the whole network is the sample
        weights = {name: qt.values for name, qt in model.weights.items()}
        from paper_2406_02629_b200.layers import plan_schedule
        from paper_2406_02629_b200.model import random_input
        from paper_2406_02629_b200.sss import SssScheme
        from paper_2406_02629_b200.field import PrimeField
        ops, _ = plan_schedule(model, SssScheme(PrimeField(), k, n), verify=verify)
        x = random_input(1, model, 0)[0]
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < budget_s / 4 or reps == 0:
            sim.simulate([op.meta() for op in ops], sim.Scheme(k, n), 7, x, weights, verify=verify)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        return {"value": 1.0 / dt, "unit": "images/s", "cores": cores, "kind": "port",
                "sample": f"oracle/sim.py full {n}PC protocol, 1 image x {reps}", "s_per_image": dt}
    weights = model.weight_values()
    total_macs = model.macs()
    # residual nets: one representative residual block (the network's most repeated kind),
    # run as its own schedule through the full protocol, extrapolated by field-MAC share
    ops = _flag_passive(model.plan_ops(), verify)
    names = [op.name for op in ops]
    stage = max({nm.split(".")[0] for nm in names if nm.startswith("s")},
                key=lambda s: sum(1 for nm in names if nm.startswith(s + ".")))
    blk = f"{stage}.b1"
    idx = [i for i, op in enumerate(ops) if op.name.startswith(blk + ".") or op.name.startswith("div." + blk + ".")]
    first, last = idx[0], idx[-1]
    remap = {i: j for j, i in enumerate(idx)}
    block_in = (first - 1) if ops[first].src is None else ops[first].src
    sub = []
    for i in idx:
        op = ops[i]
        s = i - 1 if op.src is None else op.src
        src = -1 if s == block_in else remap[s]
        kw = {"src": src if src != remap.get(i, 0) - 1 else None}
        if op.kind == "add":
            s2 = op.src2
            kw["src2"] = -1 if s2 == block_in else remap[s2]
        sub.append(op.replace(**kw))
    sub.append(ScheduledOp("output", -1, "output", ops[last].out_shape, ops[last].out_shape))
    sub = _flag_passive(sub, verify)
    blk_macs = 0
    for op in sub:
        if op.kind == "linear":
            w = weights[op.weight + ".w"]
            blk_macs += int(np.prod(op.out_shape)) * int(np.prod(w.shape[1:]))
    rng = np.random.default_rng(1)
    x = rng.integers(0, 1 << 10, size=tuple(ops[first].in_shape))
    t0 = time.perf_counter()
    sim.simulate([op.meta() for op in sub], sim.Scheme(k, n), 7, x, weights, verify=verify)
    dt = time.perf_counter() - t0
    s_per_img = dt * total_macs / blk_macs
    return {"value": 1.0 / s_per_img, "unit": "images/s", "cores": cores, "kind": "port",
            "sample": (f"oracle/sim.py lockstep {n}PC protocol (C arithmetic, OpenMP) on residual block {blk} "
                       f"({len(sub) - 1} ops, {blk_macs / 1e9:.3f} of {total_macs / 1e9:.2f} GMAC) for 1 image: "
                       f"{dt:.1f} s, extrapolated by field-MAC share"),
            "s_per_image": s_per_img}


def load_traffic(workload=None):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged per kernel class over
    one full step, from the committed ncu capture (profiles/<round>/traffic.json), or {} when the
    capture is of another workload."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic.json")))
    if not files:
        return {}
    try:
        with open(files[-1]) as fh:
            d = json.load(fh)
        if workload is not None and d.get("workload", "resnet152-5pc") != workload:
            return {}
        return d.get("bytes_per_launch", {})
    except (OSError, ValueError):
        return {}


# executed thread instructions and FMA-heavy pipe cycles (per SM, 4 pipe slots per SM per cycle) per
# chain element, by workload: ncu smsp__thread_inst_executed / sm__pipe_fmaheavy_cycles_active over the
# chain kernels of one ResNet-152 step (batch 32) / the step's chain elements (tools/chain_alu.py,
# profiles/r02/alu/).  The chain kernels are bound by the FMA-heavy pipe that executes IMAD.
CHAIN_ALU = {"resnet152-5pc": 1943, "resnet152-3pc": 1111}
CHAIN_HEAVY = {"resnet152-5pc": 64.9, "resnet152-3pc": 35.0}


def roofline(kstats, eng, dev_ms, bf16, hbm, src, workload=None):
    """Roofline of the dominant kernel class of the step (by device time), plus every class.
    gemm: int8 tensor ops = L^2 * 2 * field MACs (L = 6 u8 limbs per 45-bit share) against the
    int8 peak, 2 x measured dense bf16 (sustained: the GEMM runs inside a long step).
    chain / im2col: algorithmic HBM bytes against the measured copy bandwidth."""
    traffic = load_traffic(workload)
    L2 = eng.limb_products()
    i8 = measured_int8()
    if i8:                       # measured int8 tensor peak (sustained: the GEMM runs inside a long step)
        peak_int8, peak_burst = i8["sustained"], i8["burst"]
        peak_note = f"peak = measured sustained dense int8 ({i8['src']}: back-to-back tcgen05.mma.kind::i8)"
    else:
        peak_int8, peak_burst = 2.0 * bf16, 2.0 * burst_bf16()
        peak_note = f"peak = 2 x {src} dense bf16 ({bf16} TF/s, sm_100 int8 MMA rate is 2x bf16)"
    rows = {}
    for cls, st in kstats.items():
        if not st["launches_per_step"] or cls == "gemm_simt":
            continue
        sec = st["ms_per_launch"] / 1e3
        if cls == "gemm":
            achieved = 2.0 * L2 * st["work_per_launch"] / sec / 1e12
            r = {"bound": "tensor", "achieved": round(achieved, 1), "peak": round(peak_int8, 1), "unit": "TFLOP/s",
                 "frac": round(achieved / peak_int8, 4),
                 "frac_vs_burst_peak": round(achieved / peak_burst, 4),
                 "field_gops": round(2.0 * st["work_per_launch"] / sec / 1e9, 1),
                 "note": f"int8 ops = {L2} u8 limb products x 2 x field MACs; {peak_note}"}
        else:
            achieved = st["work_per_launch"] / sec / 1e9
            r = {"bound": "hbm", "achieved": round(achieved, 1), "peak": round(hbm, 1), "unit": "GB/s",
                 "frac": round(achieved / hbm, 4),
                 "note": "algorithmic bytes per launch (DESIGN.md section 3) / CUDA-event launch time"}
            alu = CHAIN_ALU.get(workload) if cls == "chain" else None      # calibrated per workload
            if alu and st.get("elems_per_launch"):
                # the fused protocol chain is integer-ALU bound: executed thread instructions per
                # element (ncu, profiles/r01/README.md) x elements / time vs the SM issue peak
                rate = alu * st["elems_per_launch"] / sec
                peak_i = 148 * 128 * 1.965e9
                r["alu_issue"] = {"thread_instr_per_elem": alu,
                                  "calibration": "ncu count, tools/chain_alu.py on this workload (batch 32)",
                                  "achieved_tinstr_per_s": float(f"{rate:.4g}"),
                                  "peak_tinstr_per_s": float(f"{peak_i:.4g}"), "frac": round(rate / peak_i, 4)}
                hv = CHAIN_HEAVY.get(workload)
                if hv:
                    # FMA-heavy pipe: hv SM-cycles per element (4 slots per SM per cycle) vs 148 SMs x clock
                    hrate = hv * st["elems_per_launch"] / sec
                    peak_h = 148 * 4 * 1.965e9
                    r["fma_heavy_pipe"] = {"slot_cycles_per_elem": hv, "achieved_per_s": float(f"{hrate:.4g}"),
                                           "peak_per_s": float(f"{peak_h:.4g}"), "frac": round(hrate / peak_h, 4),
                                           "note": "the chain's binding pipe (IMAD / IMAD.WIDE)"}
        t = traffic.get(cls)
        r["traffic"] = round(t) if t else None
        r["kernel"] = st["kernel"]
        r["launches_per_step"] = round(st["launches_per_step"], 1)
        r["ms_per_step"] = round(st["ms_per_step"], 3)
        r["share_of_step"] = round(st["ms_per_step"] / dev_ms, 4)
        r["work_per_launch"] = st["work_per_launch"]
        rows[cls] = r
    if not rows:
        return None, {}
    dom = max(rows, key=lambda c: rows[c]["ms_per_step"])
    return dict(rows[dom], kernel_class=dom), rows


def reference_cpu_baseline(model, k, n):
    """The unmodified reference (baseline/_ref) timed once on this host: one full run for chain
    models, per-op sampling for residual nets (bench_reference.py).  None if not installed."""
    import bench_reference as br
    ssnet, why = br.load_reference()
    if ssnet is None:
        return None, why
    s_img, wall, text, rows = br.reference_step(ssnet, model, k, n)
    return {"value": 1.0 / s_img, "unit": "images/s", "cores": 1, "kind": "reference",
            "sample": text + "; pure Python object arithmetic under the GIL (n+1 threads, one core busy)",
            "s_per_image": s_img, "sampling_wall_s": round(wall, 2), "per_op": rows}, None


def gemm_reference(args):
    """Reference arm of config 5: the reference's own share-GEMM expression `(w @ x) % p` on
    numpy object arrays (S/layers.py:252-254, baseline/_ref), a 96^3 sample per step; the C
    oracle port (OpenMP, all host threads) on 512^3 is reported beside it."""
    import bench_reference as br
    import oracle
    oracle.build()
    cores = oracle.set_threads(0)
    rng = np.random.default_rng(0)
    p = oracle.DEFAULT_PRIME
    S = 512
    a = rng.integers(0, p, size=(S, S), dtype=np.int64)
    b = rng.integers(0, p, size=(S, S), dtype=np.int64)
    t0 = time.perf_counter()
    oracle.gemm(a, b, p)
    port = 2.0 * S ** 3 / (time.perf_counter() - t0) / 1e9
    ssnet, why = br.load_reference()
    vals, walls = [], []
    for _ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if ssnet is not None:
            rate, RS = br.gemm_rate(ssnet)
            vals.append(rate / 1e9)
        else:
            oracle.gemm(a, b, p)
            vals.append(2.0 * S ** 3 / (time.perf_counter() - t0) / 1e9)
        walls.append(time.perf_counter() - t0)
    v = float(np.median(vals[args.warmup:] or vals))
    wall_ms = float(np.median(walls[args.warmup:] or walls)) * 1e3
    if ssnet is not None:
        cb = {"value": round(v, 4), "unit": "Gop/s", "cores": 1, "kind": "reference",
              "sample": f"reference (w @ x) % p on {RS}^3 numpy object arrays (baseline/_ref); rate is size-independent"}
    else:
        cb = {"value": round(v, 4), "unit": "Gop/s", "cores": cores, "kind": "port",
              "sample": f"oracle C exact mod-p GEMM {S}^3 (reference unavailable: {why})"}
    cb["port"] = {"value": round(port, 3), "unit": "Gop/s", "cores": cores, "kind": "port",
                  "sample": f"oracle/ssn_oracle.c exact mod-p GEMM {S}^3 (u128 accumulate, OpenMP)"}
    return {"metric": "mod-p share GEMM field Gop/s (largest sweep shape, summed over GPUs)", "value": round(v, 4),
            "unit": "Gop/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(wall_ms, 1), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (uniform field elements)",
            "config": {"workload": "gemm-sweep"}, "cpu_baseline": cb,
            "e2e": {"value": round(v, 4), "unit": "Gop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_reference(args):
    """--impl reference: the unmodified reference package through its own API
    (bench_reference.py), rank 0 only; each step is a bounded sample (a full run for chain
    models, per-op sampling for residual nets) and ms_per_step is the time it really took."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.workload == "gemm-sweep":
        print(json.dumps(gemm_reference(args)), flush=True)
        return
    import bench_reference as br
    name = WORKLOADS[args.workload]
    model = build_model(name[0])
    k, n, verify = name[1], name[2], name[3]
    ssnet, why = br.load_reference()
    s_img, walls, text, rows = [], [], None, None
    for _ in range(args.warmup + args.steps):
        if ssnet is not None:
            si, wall, text, rows = br.reference_step(ssnet, model, k, n)
        else:
            t0 = time.perf_counter()
            port = cpu_baseline_sample(model, k, n, verify, budget_s=args.cpu_budget)
            si, wall, text = port["s_per_image"], time.perf_counter() - t0, port["sample"] + f" (reference unavailable: {why})"
        s_img.append(si)
        walls.append(wall)
    si = float(np.median(s_img[args.warmup:] or s_img))
    wall_ms = float(np.median(walls[args.warmup:] or walls)) * 1e3
    v = 1.0 / si
    if ssnet is not None:
        cb = {"value": v, "unit": "images/s", "cores": 1, "kind": "reference",
              "sample": text + "; pure Python object arithmetic under the GIL (n+1 threads, one core busy)",
              "s_per_image": si, "per_op": rows}
        try:
            cb["port"] = cpu_baseline_sample(model, k, n, verify, budget_s=args.cpu_budget)
        except Exception as exc:
            cb["port"] = {"error": repr(exc)}
    else:
        cb = {"value": v, "unit": "images/s", "cores": port["cores"], "kind": "port", "sample": text, "s_per_image": si}
    out = {"metric": metric_for(args.workload), "value": v, "unit": "images/s", "impl": "reference",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(wall_ms, 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
           "data": "synthetic", "config": {"workload": args.workload, "k": k, "n": n, "verify": False,
                                           "batch_per_step": 1, "s_per_image": si,
                                           "note": ("ms_per_step is the wall time of one step's bounded sample; "
                                                    "value is the reference's images/s extrapolated from it "
                                                    "(bench_reference.py). The reference has no verification step.")},
           "cpu_baseline": cb,
           "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_gemm_sweep(args):
    """Config 5: one party's mod-p share GEMM C = A.B^T over uniform field elements (u8 limb
    planes, tcgen05) for M,N,K in SWEEP, plus the reshare microbenchmark (reshare_microbench:
    co-resident R^T apply against HBM, and at >= 2 GPUs one all-pairs NCCL hop against NVLink).  Every rank runs the sweep on its own GPU (weak scaling, no collective); value =
    summed field Gop/s of the largest shape.  Exactness: a 256^3 slice against the CUDA-core
    reference GEMM (ssn_dense_simt)."""
    import torch
    import torch.distributed as dist
    from paper_2406_02629_b200 import _lib, gemm as G
    from paper_2406_02629_b200.field import PrimeField
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p = PrimeField().p
    L = G.limbs(p)
    hbm, _, _ = measured_peaks()
    # GEMMs timed alone, back to back -> the burst bf16 figure (B200_PROFILING.md)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            bf16, src = json.load(fh)["bf16_tflops"], "measured burst"
    except (OSError, KeyError, ValueError):
        bf16, src = 1590.0, "fallback"
    peak = 2.0 * bf16
    i8 = measured_int8()
    if i8:                                  # GEMMs timed alone: the measured burst int8 figure
        peak, src = i8["burst"], f"measured burst dense int8 ({i8['src']})"
    st = torch.cuda.current_stream()

    def rand_field(n, stream_id):
        t = torch.empty(n, dtype=torch.int64, device="cuda")
        _lib.call("ssn_rand", _lib.ptr(t), n, 0, p, 1234 + rank, stream_id, _lib.stream_ptr())
        return t

    def planes_of(x, rows, K):
        pl = torch.empty((L, rows, G.kpad(K)), dtype=torch.uint8, device="cuda")
        _lib.call("ssn_limb_split", _lib.ptr(x), rows, K, G.kpad(K), L, _lib.ptr(pl), rows * K, 1, _lib.stream_ptr())
        return pl

    # exactness gate: tensor-core vs CUDA-core GEMM on 256^3
    a = rand_field(256 * 256, 1).reshape(256, 256)
    b = rand_field(256 * 256, 2).reshape(256, 256)
    ref = torch.empty((256, 256), dtype=torch.int64, device="cuda")     # [img=m][o=n]
    _lib.call("ssn_dense_simt", _lib.ptr(b), 0, _lib.ptr(a), 0, _lib.ptr(ref), 0, 1, 256, 256, 256, p,
              _lib.stream_ptr())
    tc = G.field_matmul(planes_of(a, 256, 256), planes_of(b, 256, 256), 256, 256, 256, p)   # [n][m]
    exact = bool(torch.equal(tc.t(), ref))
    rows = []
    sampler = ClockSampler(local)
    sampler.start()
    for (M, N, K) in SWEEP:
        A = planes_of(rand_field(M * K, 3), M, K)
        Bp = planes_of(rand_field(N * K, 4), N, K)
        out = torch.empty((N, M), dtype=torch.int64, device="cuda")
        for _ in range(max(1, args.warmup)):
            G.field_matmul(A, Bp, M, N, K, p, out=out)
        torch.cuda.synchronize()
        reps = max(1, args.steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = _lib.launch_count()
        e0.record(st)
        for _ in range(reps):
            G.field_matmul(A, Bp, M, N, K, p, out=out)
        e1.record(st)
        torch.cuda.synchronize()
        launches = (_lib.launch_count() - l0) // reps
        sec = e0.elapsed_time(e1) / reps / 1e3
        fops = 2.0 * M * N * K / sec
        rows.append({"M": M, "N": N, "K": K, "ms": round(sec * 1e3, 3), "field_gops": round(fops / 1e9, 1),
                     "int8_tops": round(L * L * fops / 1e12, 1), "frac_int8": round(L * L * fops / 1e12 / peak, 4),
                     "split_k": G.kpad(K) > G.max_k_chunk(p)})
        del A, Bp, out
    clocks = sampler.stop()
    top = rows[-1]
    value = top["field_gops"]
    # exactness at the headline shape (split-K): a 256 x 256 output block of the 16384^3 GEMM
    # against the CUDA-core GEMM on the same rows/columns
    M, N, K = SWEEP[-1]
    Ah, Bh = rand_field(M * K, 5).reshape(M, K), rand_field(N * K, 6).reshape(N, K)
    big = G.field_matmul(planes_of(Ah, M, K), planes_of(Bh, N, K), M, N, K, p)      # [n][m]
    blk = torch.empty((256, 256), dtype=torch.int64, device="cuda")
    a_blk, b_blk = Ah[:256].contiguous(), Bh[:256].contiguous()
    _lib.call("ssn_dense_simt", _lib.ptr(b_blk), 0, _lib.ptr(a_blk), 0, _lib.ptr(blk), 0, 1, 256, 256, K, p,
              _lib.stream_ptr())
    exact_top = bool(torch.equal(big[:256, :256].t(), blk))
    del big, blk
    # end to end through the public API (gemm.field_matmul) with host buffers: pinned u64 field
    # elements in, limb split + tcgen05 GEMM on the device, the u64 product back to the host
    A_host, B_host = Ah.cpu().pin_memory(), Bh.cpu().pin_memory()
    del Ah, Bh
    C_host = torch.empty((N, M), dtype=torch.int64).pin_memory()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def e2e_step():
        a_d = A_host.to("cuda", non_blocking=True)
        b_d = B_host.to("cuda", non_blocking=True)
        c_d = G.field_matmul(planes_of(a_d, M, K), planes_of(b_d, N, K), M, N, K, p)
        C_host.copy_(c_d, non_blocking=True)
    e2e_step()
    torch.cuda.synchronize()
    ee0.record(st)
    for _ in range(max(1, args.steps)):
        e2e_step()
    ee1.record(st)
    torch.cuda.synchronize()
    e2e_s = ee0.elapsed_time(ee1) / max(1, args.steps) / 1e3
    e2e = {"value": round(2.0 * M * N * K / e2e_s / 1e9, 1), "unit": "Gop/s",
           "h2d_bytes_per_step": int(A_host.numel() * 8 + B_host.numel() * 8), "d2h_bytes_per_step": int(C_host.numel() * 8)}
    del A_host, B_host, C_host
    reshare = reshare_microbench(args, torch, dist, _lib, p, hbm, world, rank)
    if world > 1:
        t = torch.tensor([value], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        value = float(t.item())
    if rank == 0:
        line = {"metric": "mod-p share GEMM field Gop/s (largest sweep shape, summed over GPUs)",
                "value": round(value, 1), "unit": "Gop/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": top["ms"], "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic (uniform field elements)",
                "config": {"workload": "gemm-sweep", "shapes": [list(r) for r in SWEEP], "limbs": L,
                           "int8_products_per_field_mac": L * L},
                "roofline": {"bound": "tensor", "achieved": top["int8_tops"], "peak": round(peak, 1),
                             "unit": "TFLOP/s", "frac": top["frac_int8"], "traffic": None,
                             "note": f"peak = {src}" if i8 else f"peak = 2 x {src} dense bf16"},
                "gpu_launches": int(launches), "exact_vs_cuda_core_gemm": exact,
                "exact_headline_block_vs_cuda_core_gemm": exact_top, "sweep": rows,
                "reshare": reshare, "clocks": clocks, "e2e": e2e}
        if not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = gemm_reference(argparse.Namespace(warmup=0, steps=1, gpus=1))["cpu_baseline"]
            except Exception as exc:
                line["cpu_baseline"] = {"value": None, "error": repr(exc)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


NVLINK_GBPS = 900.0          # NVLink 5 per direction per GPU (B200_PROFILING.md / datasheet)


def reshare_microbench(args, torch, dist, _lib, p, hbm, world, rank):
    """Config 5's reshare half.  (a) Co-resident: step 2 of reshare_degree_reduce
    (S/protocol.py:165-185) on a 4096^2 GEMM output of the (3,5) scheme -- each of the k front
    ranks applies R^T to the m = 5 participants' sub-shares (ssn_reduce_apply), algorithmic bytes
    8*(m + n) per element per front rank, against HBM.  (b) Party-per-GPU (world >= 2): one
    reshare hop's traffic, every rank sending a 4096^2-element share buffer to every other rank
    at once (NCCL send/recv in one group), max-over-ranks time, per-rank egress against NVLink."""
    from paper_2406_02629_b200.field import PrimeField
    from paper_2406_02629_b200.sss import SssScheme
    k, n = 3, 5
    m = 2 * k - 1
    sch = SssScheme(PrimeField(), k, n)
    R = sch.reducing_matrix()
    rt = _lib.u64_array([R[j][t] for t in range(n) for j in range(m)])
    E = 4096 * 4096
    sub = torch.empty((k, m, E), dtype=torch.int64, device="cuda")
    _lib.call("ssn_rand", _lib.ptr(sub), sub.numel(), 0, p, 99 + rank, 7, _lib.stream_ptr())
    back = torch.empty((k, n, E), dtype=torch.int64, device="cuda")

    def apply():
        _lib.call("ssn_reduce_apply", _lib.ptr(sub), m * E, E, m, rt, n, _lib.ptr(back), n * E, E, E, k, p,
                  _lib.stream_ptr())
    for _ in range(max(1, args.warmup)):
        apply()
    reps = max(1, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        apply()
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / reps / 1e3
    gbs = 8.0 * (m + n) * E * k / sec / 1e9
    out = {"coresident_reduce_apply": {"scheme": [k, n], "elements": E, "front_ranks": k,
                                       "ms": round(sec * 1e3, 3), "achieved_GBps": round(gbs, 1),
                                       "peak_GBps": round(hbm, 1), "frac_hbm": round(gbs / hbm, 4),
                                       "bytes_per_elem_per_front": 8 * (m + n)}}

    def timed(fn, nbytes):
        for _ in range(max(1, args.warmup)):
            fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t_s = e0.elapsed_time(e1) / reps / 1e3
        return {"ms": round(t_s * 1e3, 3), "achieved_GBps": round(nbytes / t_s / 1e9, 1),
                "frac_hbm": round(nbytes / t_s / 1e9 / hbm, 4)}
    # step 1 / SHARE_DIST: gen of n shares from a secret, Philox coefficients in registers
    ids = _lib.u64_array(list(sch.party_ids))
    sec_in = sub[0, 0]
    gen_out = back[0]
    out["gen"] = dict(timed(lambda: _lib.call("ssn_gen", _lib.ptr(sec_in), E, None, 0, 5, 11, k - 1, ids, n,
                                              _lib.ptr(gen_out), n * E, E, E, 1, p, _lib.stream_ptr()),
                            8.0 * (1 + n) * E), bytes_per_elem=8 * (1 + n), ids=n)
    # step 3 / elite reconstruction: rec over the k front ranks
    wf = _lib.u64_array(list(sch.lagrange_weights(sch.front_ids)))
    rec_out = back[1, 0]
    out["rec"] = dict(timed(lambda: _lib.call("ssn_rec", _lib.ptr(sub[0]), 0, E, wf, k, _lib.ptr(rec_out), 0, E, 1, p,
                                              _lib.stream_ptr()), 8.0 * (k + 1) * E), bytes_per_elem=8 * (k + 1))
    # truncation elite (S/layers.py:295-315): rec over the fronts, RS check of the n-k extra masked
    # shares, window decode / floor / round, fresh (k, n) shares
    from paper_2406_02629_b200.protocol import extrapolation_coeffs
    ext = _lib.u64_array([v for row in extrapolation_coeffs(sch, sch.front_ids, sch.party_ids[k:]) for v in row])
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    masked = back[0]
    tr_out = sub[1]
    out["trunc_elite"] = dict(timed(lambda: _lib.call(
        "ssn_trunc_elite", _lib.ptr(masked), E, n, k, wf, ext, 1 << 40, 1 << 12, 1, None, 5, 13, k - 1, ids, n,
        _lib.ptr(tr_out), E, _lib.ptr(fail), E, p, _lib.stream_ptr()), 8.0 * (n + n) * E),
        bytes_per_elem=8 * (n + n), rs_checks=n - k)
    # nonlinear elite (S/layers.py:345-364): rec over the 2k-1 participants, decode, ReLU, encode
    wp = _lib.u64_array(list(sch.lagrange_weights(sch.participating_ids)))
    plain = sub[2, 0]
    out["nonlin_elite"] = dict(timed(lambda: _lib.call(
        "ssn_nonlin_elite", _lib.ptr(back[1]), E, m, wp, 1, 0, 1, 1, 4096, 4096, 1, 1, _lib.ptr(plain), p,
        _lib.stream_ptr()), 8.0 * (m + 1) * E), bytes_per_elem=8 * (m + 1))
    del sub, back
    if world < 2:
        out["exchange"] = {"unavailable": "party-per-GPU exchange needs >= 2 GPUs"}
        return out
    Ex = 4096 * 4096
    send = [torch.empty(Ex, dtype=torch.int64, device="cuda") for _ in range(world)]
    recv = [torch.empty(Ex, dtype=torch.int64, device="cuda") for _ in range(world)]

    def hop():
        ops = []
        for peer in range(world):
            if peer != rank:
                ops.append(dist.P2POp(dist.isend, send[peer], peer))
                ops.append(dist.P2POp(dist.irecv, recv[peer], peer))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    dist.barrier()
    for _ in range(max(1, args.warmup)):
        hop()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for _ in range(reps):
        hop()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t.item()) / 1e3
    egress = 8.0 * Ex * (world - 1) / sec / 1e9
    out["exchange"] = {"ranks": world, "elements_per_peer": Ex, "ms": round(sec * 1e3, 3),
                       "egress_GBps_per_rank": round(egress, 1), "peak_GBps": NVLINK_GBPS,
                       "frac_nvlink": round(egress / NVLINK_GBPS, 4)}
    return out


def run_party_placement(args):
    """Party-per-GPU placement (sharded.PartyShardedEngine): ranks [g*(n+1), (g+1)*(n+1)) form
    group g (trusted source + n parties, elite rotating over the front ranks); the GPUs no group
    uses each run a co-resident replica (all n parties on one GPU, its own batch) so no GPU
    idles.  value = (G*B + L*B_co) images / max-over-ranks step time."""
    import torch
    import torch.distributed as dist
    from paper_2406_02629_b200 import _lib, resnet
    from paper_2406_02629_b200.batched import BatchedEngine, StreamPipelinedEngine
    from paper_2406_02629_b200.field import PrimeField
    from paper_2406_02629_b200.sharded import PartyShardedEngine
    from paper_2406_02629_b200.sss import SssScheme
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SSN_SHARED_GPU=1: every rank on cuda:0 with host-staged gloo (single-GPU functional check)
    shared = os.environ.get("SSN_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    kind, k, n, verify, dflt_batch = WORKLOADS[args.workload]
    groups = world // (n + 1)
    leftover = world - groups * (n + 1)
    if groups < 1:
        if rank == 0:
            print(json.dumps({"metric": metric_for(args.workload), "unavailable":
                              f"party placement needs >= n+1 = {n + 1} GPUs, got {world}"}), flush=True)
        return
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B = args.batch or dflt_batch
    model = build_model(kind)
    scheme = SssScheme(PrimeField(), k, n)
    g = rank // (n + 1)
    in_group = g < groups
    if in_group:
        eng = PartyShardedEngine(model, scheme, batch=B, seed=7 + g, verify=verify, group=g)
    else:                                   # a leftover GPU: co-resident replica
        ns = DEFAULT_STREAMS.get(args.workload, 1)
        eng = (StreamPipelinedEngine(model, scheme, batch=B, streams=ns, seed=7 + rank, verify=verify) if ns > 1
               else BatchedEngine(model, scheme, batch=B, seed=7 + rank, verify=verify))
        for e in getattr(eng, "engines", [eng]):
            e.defer_verify = True
    # a collective before the first point-to-point call creates the NCCL communicator on every
    # rank (batch_isend_irecv as the first call of a group must otherwise involve all ranks)
    dist.barrier()
    xb = (model.random_inputs(seed=100 + rank, batch=B) if hasattr(model, "random_inputs")
          else np.stack([__import__("paper_2406_02629_b200.model", fromlist=["random_input"])
                         .random_input(100 + rank, model, index=i)[0] for i in range(B)]))
    if in_group:
        xb = (model.random_inputs(seed=100 + g, batch=B) if hasattr(model, "random_inputs") else xb)
    x_dev = torch.as_tensor(xb, device="cuda")
    outputs_match = None
    if not args.no_check:
        got = eng.run(xb)
        if (not in_group or eng.role == 1) and hasattr(model, "nodes"):
            want = resnet.plaintext_forward(model, xb, device="cuda")[0]
            outputs_match = bool(np.array_equal(got, want))
    for _ in range(args.warmup):
        eng.run_device(x_dev)
    torch.cuda.synchronize()
    dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    e0.record()
    for _ in range(args.steps):
        eng.run_device(x_dev)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    cdev = "cpu" if shared else "cuda"
    nl = torch.tensor([float((_lib.launch_count() - l0) // args.steps)], dtype=torch.float64, device=cdev)
    dist.all_reduce(nl, op=dist.ReduceOp.SUM)
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    m = torch.tensor([float(outputs_match is True), float(outputs_match is not None)], device=cdev)
    dist.all_reduce(m, op=dist.ReduceOp.SUM)
    ms = float(t.item())
    checked = int(m[1].item())
    match = None if checked == 0 else int(m[0].item()) == checked
    if rank == 0:
        imgs = groups * B + leftover * B
        line = {"metric": metric_for(args.workload), "value": round(imgs / (ms / 1e3), 3), "unit": "images/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic",
                "config": {"workload": args.workload, "model": model.name, "k": k, "n": n, "verify": verify,
                           "placement": (f"party-per-GPU: {groups} group(s) x (source + {n} parties, elite rotating "
                                         f"over the {k} front ranks) + {leftover} co-resident replica GPU(s)"),
                           "batch_per_group": B, "global_batch": imgs,
                           "parallelism": f"party{n + 1} x dp{groups} + coresident x {leftover}"},
                "gpu_launches": int(nl.item()), "gpu_launches_scope": "summed over ranks, per step",
                "clocks": clocks, "outputs_match_plaintext": match}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--workload", default="resnet152-5pc", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-latency", action="store_true", help="skip the batch-1 latency measurement")
    ap.add_argument("--streams", type=int, default=None,
                    help="co-resident: split the batch over this many CUDA streams (GEMM/chain overlap)")
    ap.add_argument("--placement", default="coresident", choices=["coresident", "party"],
                    help="coresident: every GPU runs all n parties on its own batch (default); "
                         "party: one GPU per party + one for the trusted source, NCCL p2p per hop, "
                         "G = N // (n+1) groups data-parallel over images")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "gemm-sweep":
        return run_gemm_sweep(args)
    if args.placement == "party":
        return run_party_placement(args)

    import torch
    import torch.distributed as dist
    from paper_2406_02629_b200 import _lib, resnet
    from paper_2406_02629_b200.batched import BatchedEngine
    from paper_2406_02629_b200.field import PrimeField
    from paper_2406_02629_b200.sss import SssScheme

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SSN_SHARED_GPU=1: every rank on cuda:0 over gloo (functional check of the multi-rank
    # timing / reduction logic on a single-GPU box; never used for reported numbers)
    shared = os.environ.get("SSN_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if shared else "cuda"
    kind, k, n, verify, dflt_batch = WORKLOADS[args.workload]
    B = args.batch or dflt_batch
    nstreams = args.streams if args.streams is not None else DEFAULT_STREAMS.get(args.workload, 1)
    if B % nstreams:
        nstreams = 1
    model = build_model(kind)
    scheme = SssScheme(PrimeField(), k, n)
    if nstreams > 1:
        from paper_2406_02629_b200.batched import StreamPipelinedEngine
        eng = StreamPipelinedEngine(model, scheme, batch=B, streams=nstreams, seed=7 + rank, verify=verify)
    else:
        eng = BatchedEngine(model, scheme, batch=B, seed=7 + rank, verify=verify)
    shape = (B,) + tuple(model.input_shape)
    if hasattr(model, "random_inputs"):
        xb = model.random_inputs(seed=100 + rank, batch=B)
    else:
        from paper_2406_02629_b200.model import random_input
        xb = np.stack([random_input(100 + rank, model, index=i)[0] for i in range(B)])
    x_dev = torch.as_tensor(xb, device="cuda")
    x_host = torch.as_tensor(xb).pin_memory()

    # correctness gate (untimed): decoded outputs == exact integer plaintext
    outputs_match = None
    if not args.no_check:
        got = eng.run(xb)
        if hasattr(model, "nodes"):
            want, _ = resnet.plaintext_forward(model, xb, device="cuda")
        else:
            from paper_2406_02629_b200.model import plaintext_infer
            want = np.stack([plaintext_infer(model, xb[i]) for i in range(B)])
        outputs_match = bool(np.array_equal(got, want))
        if world > 1:                       # every rank's batch must match, not just rank 0's
            t = torch.tensor([float(outputs_match)], dtype=torch.float64, device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            outputs_match = bool(t.item() == 1.0)

    stream = torch.cuda.current_stream()

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        eng.run_device(x_dev)
    # verification runs in every step's kernels; its host-side failure check is deferred to the
    # end of the timed region (no per-step sync)
    for e in getattr(eng, "engines", [eng]):
        e.defer_verify = True
    # ---- device-resident timed region (value) ----
    sampler = ClockSampler(local)
    sampler.start()
    eng.enable_profiling()
    sync_all()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # per-kernel CUDA events are recorded on the first timed step only (inside the timed region;
    # ~600 event pairs per step would otherwise cost about 1% of the measured time)
    engines = getattr(eng, "engines", [eng])
    prof_steps, stash = min(1, args.steps), None
    e0.record(stream)
    for i in range(args.steps):
        if i == prof_steps:
            stash = [(e, e._prof) for e in engines]
            for e in engines:
                e._prof = None
        if i < prof_steps and nstreams > 1:
            # the profiled step runs the stream sub-batches back to back, so every kernel's
            # CUDA-event time is its own (no co-running kernels); the other steps overlap
            eng.run_device(x_dev, serial=True)
        else:
            eng.run_device(x_dev)
    e1.record(stream)
    sync_all()
    if stash is not None:
        for e, pr in stash:
            e._prof = pr
    launches = (_lib.launch_count() - l0) // args.steps
    dev_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    kstats = eng.profile_summary(max(prof_steps, 1) if stash is not None else args.steps)
    eng.disable_profiling()
    clocks = sampler.stop()
    # host enqueue cost of one step with an empty launch queue (CUDA-graph rationale: it must
    # stay below the device time for the GPU never to starve); outside the timed region
    h0 = time.perf_counter()
    eng.run_device(x_dev)
    host_ms = (time.perf_counter() - h0) * 1e3
    torch.cuda.synchronize()
    verify_failures = 0
    for e in getattr(eng, "engines", [eng]):
        if e.verify:
            verify_failures += int(e.fail.item())
    if world > 1:
        t = torch.tensor([float(verify_failures)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t)
        verify_failures = int(t.item())
    # ---- end-to-end through the public API with host buffers (e2e) ----
    out_host = torch.empty((B,) + eng.out_shape(), dtype=torch.int64).pin_memory()
    sync_all()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        xd = x_host.to("cuda", non_blocking=True)
        out = eng.run_device(xd)
        out_host.copy_(out, non_blocking=True)
    t1.record(stream)
    sync_all()
    e2e_ms = max_over_ranks(t0.elapsed_time(t1) / args.steps)

    # per-op-kind breakdown from one extra instrumented step (not part of the timed region)
    breakdown = {}
    eng.run_device(x_dev, timings=breakdown)

    # batch-1 latency (the paper's per-image setting): one image, one stream,
    # device-resident input, CUDA events over `steps` back-to-back inferences
    latency = None
    if not args.no_latency:
        first = getattr(eng, "engines", [eng])[0]
        e1eng = BatchedEngine(model, scheme, batch=1, seed=7 + rank, verify=verify, share_weights_with=first)
        e1eng.defer_verify = True
        x1 = x_dev[:1].contiguous()
        for _ in range(max(args.warmup, 2)):
            e1eng.run_device(x1)
        torch.cuda.synchronize()
        l_0, l_1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nlat = max(args.steps, 5)
        l_0.record(stream)
        for _ in range(nlat):
            e1eng.run_device(x1)
        l_1.record(stream)
        torch.cuda.synchronize()
        lat_ms = l_0.elapsed_time(l_1) / nlat
        latency = {"batch": 1, "streams": 1, "steps": nlat, "ms_per_image": round(lat_ms, 3),
                   "s_per_image": round(lat_ms / 1e3, 6), "images_per_s": round(1e3 / lat_ms, 2)}
        del e1eng

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    imgs = B * world
    value = imgs / (dev_ms / 1000.0)
    e2e = imgs / (e2e_ms / 1000.0)
    hbm, bf16, src = measured_peaks()
    online, offline = eng.comm_per_image()
    roof, by_kernel = roofline(kstats, eng, dev_ms, bf16, hbm, src, workload=args.workload)
    cpu = None
    if not args.no_cpu_baseline and world == 1:          # the CPU baseline is an N=1 figure
        try:
            port = cpu_baseline_sample(model, k, n, verify, budget_s=args.cpu_budget)
        except Exception as exc:       # reported, never silently replaced
            port = {"value": None, "error": repr(exc)}
        try:
            cpu, why = reference_cpu_baseline(model, k, n)
        except Exception as exc:
            cpu, why = None, repr(exc)
        if cpu is None:
            cpu = dict(port, reference_unavailable=why)
        else:
            cpu["port"] = port
    line = {
        "metric": metric_for(args.workload), "value": round(value, 3), "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": args.workload, "model": model.name, "k": k, "n": n, "verify": verify,
                   "batch_per_gpu": B, "global_batch": imgs, "parallelism": f"dp{world} x co-resident {n} parties",
                   "rng": "device philox", "l2": "working set >> 126 MB L2 (inputs larger than L2)",
                   "streams_per_gpu": nstreams, "batch_latency_ms": round(dev_ms, 3),
                   "inverse_throughput_s_per_image": round(dev_ms / 1000.0 / B, 6)},
        "e2e": {"value": round(e2e, 3), "unit": "images/s",
                "h2d_bytes_per_step": int(x_host.numel() * 8), "d2h_bytes_per_step": int(out_host.numel() * 8)},
        "gpu_launches": int(launches),
        "host_enqueue_ms_per_step": round(host_ms, 3),
        "verification_failures": verify_failures if verify else None,
        "roofline": roof,
        "roofline_by_kernel": by_kernel,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "outputs_match_plaintext": outputs_match,
        "comm_per_image_GB": {"online": round(online * 8 / 1e9, 3), "offline_masks": round(offline * 8 / 1e9, 3)},
        "latency_batch1": latency,
        "breakdown_ms_per_step": {kk: round(v, 3) for kk, v in breakdown.items()},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
