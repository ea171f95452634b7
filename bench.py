#!/usr/bin/env python
"""Benchmark of the fused neighborhood attention hot path (libna.so) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

Workload (BASELINE.json configs[1], the one the metric is quoted on that fits
one GPU): 1-D NA, fp16, B=8 H=16 L=16384 D=64, kernel 255, dilation {1,4} x
{non-causal, causal}.  One STEP = na_fwd + na_bwd of all four variants on one
batch (every §8(a) row of SURVEY.md).  Inputs are unit-normal, seeded per
(b, h) (na_synth), resident in HBM before timing.

metric/unit: BASELINE.json's metric; `value` = effective TFLOP/s of the whole
step over all ranks, with the paper's nominal FLOP count 4*N*l*D per (b,h)
forward and 10*N*l*D backward (2.5x, FlashAttention convention);
l = 255.  Multi-GPU (torchrun): the config's B*H slices are
split across the ranks -- rank g owns the flattened slices
[g*BH/G, (g+1)*BH/G), seeded by global slice index -- so every N computes
exactly BASELINE.json's problem (strong scaling, no collective on the data
path); NCCL only gathers timings and parity errors.  Device time = CUDA
events on the launch stream, max over ranks.

`per_config` in the JSON line: every BASELINE.json config (A; B's four
variants; C at dilation 1 and 8; D; E): fwd ms and fwd+bwd ms, effective
TFLOP/s, the fractions of the tensor peak and (forward) of HBM bandwidth,
the max-abs errors of O, LSE, dQ, dK, dV on the first and the last (b,h)
slice (every token) against the fp64 oracle's exact result (and, on the
first slice, dQ/dK against the oracle's stored-O reading R12), and the
oracle's own time on those slices extrapolated to the whole config.

`--impl reference`: the arm the driver compares against is the fp64 CPU
oracle (oracle/, test infrastructure) timed on this host's cores on a
bounded sample of the same workload (tier rules).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import threading
import sys
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import na_synth  # noqa: E402

METRIC = "fused NA fwd & fwd+bwd ms, TFLOP/s vs B200 tensor peak at 1/2/4/8 GPUs"
WORKLOAD = "1-D NA fp16 B=8 H=16 L=16384 D=64 kernel=255 dilation={1,4} x {non-causal,causal}, fwd+bwd"
VARIANTS = ["B_d1", "B_d4", "B_d1_causal", "B_d4_causal"]
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def flops(cfg, fwd=True, bwd=True):
    """Nominal FLOPs for the whole batch (4 b h n l d forward)."""
    per = 4.0 * cfg.batch * cfg.heads * cfg.tokens * cfg.window * cfg.head_dim
    return (per if fwd else 0.0) + (2.5 * per if bwd else 0.0)


def algorithmic_bytes(cfg, kernel, bh=None):
    """Bytes a kernel must move at minimum: every
    tensor it reads or writes once, for `bh` (b,h) slices (default: the whole
    config).  E = elements of one [B,H,N,D] tensor."""
    bh = cfg.batch * cfg.heads if bh is None else bh
    E = bh * cfg.tokens * cfg.head_dim
    rows = bh * cfg.tokens
    s = 2 if cfg.dtype in (torch.float16, torch.bfloat16) else 4
    return {
        "fna_fwd_tc": 4 * E * s + 4 * rows,            # Q,K,V read; O write; LSE write
        "fna_fwd_simt": 4 * E * s + 4 * rows,
        "fna_bwd_pre": 2 * E * s + 12 * rows,          # O, dO, LSE read; (-LSE log2 e, D) written
        "fna_dkdv_tc": 6 * E * s + 8 * rows,           # Q,K,V,dO read; dK,dV write; LSE,D read
        "fna_dkdv_simt": 6 * E * s + 8 * rows,
        # Rank 1 fuses the preprocess into dQ: + O read, LSE read, (-LSE log2 e, D) written.
        "fna_dq_tc": (6 * E * s + 12 * rows) if len(cfg.extent) == 1 else (5 * E * s + 8 * rows),
        "fna_dq_simt": 5 * E * s + 8 * rows,
    }[kernel]


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 5 ms by an
    NVML thread while the timed region runs (nvidia-smi fallback)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.thread = None
        self.rows = []
        self.stop_flag = threading.Event()

    def _nvml_handle(self, nv):
        nv.nvmlInit()
        try:  # match the CUDA device by PCI bus id (CUDA and NVML orders can differ)
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            import pynvml as nv
            h = self._nvml_handle(nv)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def run():
                while not self.stop_flag.is_set():
                    try:
                        sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((sm, mx, ["Active" if r & b else "Not Active" for b in bits]))
                    except Exception:
                        pass
                    time.sleep(0.005)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        rows = self.rows
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join(timeout=2)
        elif self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for line in out.strip().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) != 6:
                    continue
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[2:]))
                except ValueError:
                    continue
        if not rows:
            return None
        reasons = sorted({self.NAMES[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        sm = [r[0] for r in rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in rows),
                "samples": len(rows), "reasons": reasons,
                "source": "nvml" if self.thread is not None else "nvidia-smi"}


def env_info():
    """Where the numbers were taken (report metadata)."""
    info = {"torch": torch.__version__, "cuda": torch.version.cuda, "nproc": os.cpu_count()}
    try:
        info["gpu"] = torch.cuda.get_device_name(0)
        info["sms"] = torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:
        pass
    try:
        import pynvml as nv
        nv.nvmlInit()
        d = nv.nvmlSystemGetDriverVersion()
        info["driver"] = d.decode() if isinstance(d, bytes) else d
    except Exception:
        pass
    try:
        info["git"] = subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True,
                                     text=True, timeout=5).stdout.strip() or None
    except Exception:
        info["git"] = None
    if not info.get("git"):
        try:  # gpurun snapshots have no .git: hash the product sources instead
            import hashlib
            h = hashlib.sha1()
            for root in ("paper_2403_04690_b200/csrc", "include"):
                for f in sorted(os.listdir(os.path.join(ROOT, root))):
                    h.update(open(os.path.join(ROOT, root, f), "rb").read())
            info["src_sha1"] = h.hexdigest()[:12]
        except Exception:
            pass
    return info


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def reduce_max(x: float, world: int, device: str = "cuda") -> float:
    """Max over ranks (timings: the slowest rank defines the step)."""
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_range(rank: int, world: int, bh: int) -> tuple:
    """Strong split: rank g of G owns the flattened (b,h)
    slices [g*BH/G, (g+1)*BH/G) of a config with BH = B*H slices (floor
    boundaries, so uneven counts differ by at most one; a rank may own none)."""
    return (rank * bh // world, (rank + 1) * bh // world)


def gather_rows(vals, world: int, device: str = "cuda"):
    """all_gather of one small fp64 vector per rank -> list of per-rank lists."""
    if world == 1:
        return [list(vals)]
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return [p.tolist() for p in parts]


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ native arm

class Runner:
    """Buffers and the step function for one rank's share of the workload:
    the flattened (b,h) slices shard_range(rank, world, B*H) of config B,
    passed to the library as batch 1 x heads n (only B*H enters the kernels)."""

    def __init__(self, rank: int, world: int):
        import paper_2403_04690_b200 as na
        self.na = na
        self.cfgs = [na_synth.CONFIGS[v] for v in VARIANTS]
        c = self.cfgs[0]
        self.bh = shard_range(rank, world, c.batch * c.heads)
        n = self.bh[1] - self.bh[0]
        assert n > 0, "every rank owns at least one (b,h) slice of config B"
        q, k, v, do = na_synth.make_inputs(c, device="cuda", bh_range=self.bh)
        shape = (1, n, *c.extent, c.head_dim)
        self.q, self.k, self.v, self.do = (t.view(shape) for t in (q, k, v, do))
        self.outs = []
        for cfg in self.cfgs:
            o = torch.empty(shape, dtype=c.dtype, device="cuda")
            lse = torch.empty(shape[:-1], dtype=torch.float32, device="cuda")
            grads = [torch.empty(shape, dtype=c.dtype, device="cuda") for _ in range(3)]
            pr = na.make_problem(batch=1, heads=n, extent=list(c.extent), head_dim=c.head_dim,
                                 kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
                                 is_causal=[bool(x) for x in cfg.is_causal], dtype=c.dtype)
            ws = torch.empty((na.na_bwd_workspace_size(pr) + 3) // 4, dtype=torch.float32, device="cuda")
            self.outs.append((o, lse, grads, ws))
        self.launches = 0

    def kw(self, cfg):
        return dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
                    is_causal=[bool(x) for x in cfg.is_causal])

    def step(self, q=None, k=None, v=None, do=None, sl=None):
        """All variants, fwd + bwd; `sl` = (a, b): only slices [a, b) of this
        rank's share (q..do are then those slices' views)."""
        na = self.na
        q = self.q if q is None else q
        k = self.k if k is None else k
        v = self.v if v is None else v
        do = self.do if do is None else do
        n = 0
        for cfg, outs in zip(self.cfgs, self.outs):
            o, lse, (dq, dk, dv), ws = outs
            if sl is not None:
                a, b = sl
                o, lse, dq, dk, dv = (t[:, a:b] for t in (o, lse, dq, dk, dv))
            kw = self.kw(cfg)
            na.na_fwd(q, k, v, out=o, lse=lse, **kw)
            n += na.last_launch_count()
            na.na_bwd(q, k, v, o, do, lse, dq=dq, dk=dk, dv=dv, workspace=ws, **kw)
            n += na.last_launch_count()
        self.launches = n
        return n

    def fwd_only(self):
        for cfg, (o, lse, _, _) in zip(self.cfgs, self.outs):
            self.na.na_fwd(self.q, self.k, self.v, out=o, lse=lse, **self.kw(cfg))


def timed_steps(fn, steps, flush=None):
    """Per-step CUDA-event device time (ms) on the current stream; the L2
    flush between steps is outside the event pair."""
    st = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for a, b in evs:
        if flush is not None:
            flush.zero_()
        a.record(st)
        fn()
        b.record(st)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def oracle_sample(tokens: int, n_slices: int):
    """Inputs + step function for the fp64 oracle on a bounded sample of the
    workload: n_slices (b,h) slices of the B_d1 variant (k=255, D=64) cut to
    their first `tokens` tokens, fwd (nar_fwd) + bwd (nar_bwd)."""
    import oracle
    base = na_synth.CONFIGS["B_d1"]
    cfg = na_synth.small_config([tokens], list(base.kernel_size), list(base.dilation),
                                list(base.is_causal), head_dim=base.head_dim, batch=1,
                                heads=n_slices, dtype=base.dtype)
    q, k, v, do = na_synth.make_inputs(cfg)
    p = oracle.make_problem(1, n_slices, [tokens], cfg.head_dim, list(cfg.kernel_size),
                            list(cfg.dilation), [int(c) for c in cfg.is_causal])

    def step():
        oracle.fwd(p, q, k, v)
        oracle.bwd(p, q, k, v, do)

    fl = 14.0 * n_slices * tokens * cfg.window * cfg.head_dim
    desc = (f"{n_slices} (b,h) slices x first {tokens} tokens of B_d1 (k=255, D=64, fp16 "
            f"inputs upcast), fwd+bwd in fp64")
    return step, fl, desc


def cpu_baseline_sample():
    import oracle
    cores = oracle.num_threads()
    step, fl, desc = oracle_sample(6144, cores)
    t0 = time.perf_counter()
    step()
    dt = time.perf_counter() - t0
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
            "sample": desc + f"; {dt:.1f} s", "seconds": round(dt, 2)}


PER_CONFIG = ["A", "B_d1", "B_d1_causal", "B_d4", "B_d4_causal", "C_d1", "C_d8", "D_d2", "E"]
# per checked slice: checked, O, LSE, dQ, dK, dV, excess O/dQ/dK/dV, oracle fwd s, oracle bwd s
_SLICE_FIELDS = 12


def slice_check(cfg, host, dev_out, li, stored: bool):
    """Every token of one (b,h) slice: GPU outputs vs the fp64 oracle's exact
    forward and gradient (oracle timed while it runs); with `stored`, also
    dQ/dK against the oracle's stored-O gradient (reading R12).
    host: the slice's q, k, v, do on the host, shaped [1, X..., D]."""
    import na_tol
    import oracle
    p = oracle.make_problem(1, 1, list(cfg.extent), cfg.head_dim, list(cfg.kernel_size),
                            list(cfg.dilation), [int(c) for c in cfg.is_causal])
    hq, hk, hv, hdo = host
    t0 = time.perf_counter()
    ro, rlse = oracle.fwd_full_tokens(p, hq, hk, hv)
    t1 = time.perf_counter()
    rdq, rdk, rdv = oracle.bwd_gather(p, hq, hk, hv, hdo)
    t2 = time.perf_counter()
    o, lse, dq, dk, dv = (t[0, li].float().cpu().numpy() for t in dev_out)
    N, D = cfg.tokens, cfg.head_dim
    dt = cfg.dtype
    ref = [ro.reshape(N, D), rdq.reshape(N, D), rdk.reshape(N, D), rdv.reshape(N, D)]
    got = [o.reshape(N, D), dq.reshape(N, D), dk.reshape(N, D), dv.reshape(N, D)]
    row = [1.0, na_tol.max_abs(got[0], ref[0]), na_tol.max_abs(lse.reshape(N), rlse.reshape(N))]
    row += [na_tol.max_abs(g, r) for g, r in zip(got[1:], ref[1:])]
    row += [na_tol.excess(g, r, dt) for g, r in zip(got, ref)]
    row += [t1 - t0, t2 - t1]
    st = [0.0, 0.0]
    if stored:
        sdq, sdk, _ = oracle.bwd_gather(p, hq, hk, hv, hdo, stored_o=True)
        st = [na_tol.max_abs(got[1], sdq.reshape(N, D)), na_tol.max_abs(got[2], sdk.reshape(N, D))]
    return row, st


def per_config_table(args, world, rank, peaks):
    """Every BASELINE.json config: fwd ms and fwd+bwd ms
    (CUDA events, L2 flushed before each call, max over ranks), effective
    TFLOP/s with the paper's nominal FLOPs, the fractions of the B200 tensor
    peak and (forward) of HBM bandwidth, the kernels' parity on the first and
    last (b,h) slice, and the oracle's time on them, extrapolated.  Strong
    split: rank g owns slices shard_range(g, G, B*H) of each config."""
    import paper_2403_04690_b200 as na
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    peak_tf = float(peaks.get("bf16_tflops", 1590.0))
    peak_bw = float(peaks["hbm_gbs"])
    out = {}
    n_it = max(3, min(args.steps, 10))
    for name in PER_CONFIG:
        cfg = na_synth.CONFIGS[name]
        BH = cfg.batch * cfg.heads
        bh0, bh1 = shard_range(rank, world, BH)
        n = bh1 - bh0
        kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
                  is_causal=[bool(c) for c in cfg.is_causal])
        f_ms = fb_ms = 0.0
        rows = [[0.0] * _SLICE_FIELDS, [0.0] * _SLICE_FIELDS]
        st = [0.0, 0.0]
        impl = None
        pick = [0, 0, 0]
        if n > 0:
            shape = (1, n, *cfg.extent, cfg.head_dim)
            q, k, v, do = (t.view(shape) for t in
                           na_synth.make_inputs(cfg, device="cuda", bh_range=(bh0, bh1)))
            o = torch.empty_like(q)
            lse = torch.empty(shape[:-1], dtype=torch.float32, device="cuda")
            dq, dk, dv = (torch.empty_like(q) for _ in range(3))
            pr = na.make_problem(1, n, list(cfg.extent), cfg.head_dim, **kw, dtype=cfg.dtype)
            impl = {na.NA_IMPL_TC: "tc", na.NA_IMPL_SIMT: "simt"}.get(na.na_selected_impl(pr))
            if cfg.dtype == torch.bfloat16 and impl == "tc":  # DESIGN.md R13 variant
                impl += "-bf16-precise" if na.na_bf16_precise(pr) == 1 else "-bf16-plain"
            ws = torch.empty((na.na_bwd_workspace_size(pr) + 3) // 4, dtype=torch.float32, device="cuda")

            def fwd():
                na.na_fwd(q, k, v, out=o, lse=lse, **kw)

            def fwd_bwd():
                fwd()
                na.na_bwd(q, k, v, o, do, lse, dq=dq, dk=dk, dv=dv, workspace=ws, **kw)

            # tile-plan tuning (setup, untimed): rank 0 measures the planner's
            # candidates, every rank uses its picks (rank 0 decides)
            if rank == 0:
                pick = list(na.na_tune(q, k, v, do, **kw))
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor(pick, dtype=torch.int32, device="cuda")
            dist.broadcast(t, 0)
            pick = t.tolist()
        if n > 0:
            na.na_set_plan_choice(pr, pick)
            for _ in range(2):
                fwd_bwd()
            torch.cuda.synchronize()
        barrier(world)
        if n > 0:
            f_ms = statistics.median(timed_steps(fwd, n_it, flush))
            fb_ms = statistics.median(timed_steps(fwd_bwd, n_it, flush))
        f_ms = reduce_max(f_ms, world)
        fb_ms = reduce_max(fb_ms, world)
        # parity of every token of the config's first and last (b,h) slice,
        # checked by the rank that owns it (outputs of the last fwd_bwd)
        if n > 0 and not args.no_parity:
            outs = (o, lse, dq, dk, dv)
            for slot, gi in enumerate(sorted({0, BH - 1})):
                if bh0 <= gi < bh1:
                    # the exact inputs the kernels saw (the device generator's values)
                    host = [t[0, gi - bh0:gi - bh0 + 1].cpu() for t in (q, k, v, do)]
                    rows[slot], s2 = slice_check(cfg, host, outs, gi - bh0, stored=(gi == 0))
                    if gi == 0:
                        st = s2
        allrows = gather_rows(rows[0] + rows[1] + st, world)
        fl_f = flops(cfg, fwd=True, bwd=False)
        fl_fb = flops(cfg)
        E = cfg.batch * cfg.heads * cfg.tokens * cfg.head_dim
        s_el = 4 if cfg.dtype == torch.float32 else 2
        fwd_bytes = 4 * E * s_el + 4 * cfg.batch * cfg.heads * cfg.tokens
        entry = {
            "fwd_ms": round(f_ms, 4), "fwd_bwd_ms": round(fb_ms, 4),
            "fwd_tflops": round(fl_f / (f_ms * 1e-3) / 1e12, 3),
            "fwd_bwd_tflops": round(fl_fb / (fb_ms * 1e-3) / 1e12, 3),
            "fwd_tensor_peak_frac": round(fl_f / (f_ms * 1e-3) / 1e12 / (world * peak_tf), 5),
            "fwd_bwd_tensor_peak_frac": round(fl_fb / (fb_ms * 1e-3) / 1e12 / (world * peak_tf), 5),
            "fwd_hbm_frac": round(fwd_bytes / (f_ms * 1e-3) / 1e9 / (world * peak_bw), 4),
            "plan_pick": pick, "impl": impl, "dtype": str(cfg.dtype).replace("torch.", ""),
        }
        checked = [r[k * _SLICE_FIELDS:(k + 1) * _SLICE_FIELDS] for r in allrows for k in range(2)]
        checked = [c for c in checked if c[0] == 1.0]
        if checked:
            mx = lambda i: max(c[i] for c in checked)
            stored = [max(r[2 * _SLICE_FIELDS + j] for r in allrows) for j in range(2)]
            excess = max(mx(6), mx(7), mx(8), mx(9))
            per_slice_f = statistics.mean(c[10] for c in checked)
            per_slice_b = statistics.mean(c[11] for c in checked)
            import oracle
            entry["parity"] = {
                "slices": sorted({0, BH - 1}), "tokens_per_slice": cfg.tokens, "vs": "oracle exact (fp64)",
                "max_abs": {"O": mx(1), "LSE": mx(2), "dQ": mx(3), "dK": mx(4), "dV": mx(5)},
                "max_abs_vs_stored_o": {"dQ": stored[0], "dK": stored[1]},
                "excess_over_bound": excess, "within_bound": excess <= 0.0,
                "bound": "max(tol, half-ulp(|ref|)), tol = 1e-2 (16-bit) / 1e-4 (fp32); LSE 2e-3 / 1e-4"}
            entry["oracle"] = {
                "fwd_s_per_slice": round(per_slice_f, 3), "bwd_s_per_slice": round(per_slice_b, 3),
                "slices_timed": len(checked), "cores": oracle.num_threads(),
                "fwd_bwd_s_whole_config": round((per_slice_f + per_slice_b) * BH, 2),
                "label": f"extrapolated x{BH} from {len(checked)} slice(s)" if BH > len(checked)
                         else "measured on the whole config"}
        out[name] = entry
        if n > 0:
            del q, k, v, do, o, lse, dq, dk, dv, ws
        torch.cuda.empty_cache()
    return out


def cp_table(args, world, rank, peaks):
    """Context parallelism (paper_2403_04690_b200/cp.py)
    at N > 1: config B_d1 with ALL its B*H slices on every rank and the
    sequence split over the ranks (owned rows + a halo of k*dil rows,
    exchanged with NCCL send/recv).  fwd and fwd+bwd ms include the halo
    exchanges; max over ranks."""
    import paper_2403_04690_b200 as na
    from paper_2403_04690_b200.cp import ContextParallel
    cfg = na_synth.CONFIGS["B_d1"]
    kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
              is_causal=[bool(c) for c in cfg.is_causal])
    cp = ContextParallel(list(cfg.extent), **kw)
    a, b = cp.split.own(rank)
    s0, e0 = cp.split.slab(rank)
    q, k, v, do = (t.view(cfg.shape())[:, :, a:b].contiguous()
                   for t in na_synth.make_inputs(cfg, device="cuda"))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    state = {}

    def fwd():
        state["o"], state["lse"], state["ctx"] = cp.forward(q, k, v)

    def fwd_bwd():
        fwd()
        cp.backward(state["ctx"], do)

    for _ in range(2):
        fwd_bwd()
    torch.cuda.synchronize()
    barrier(world)
    n_it = max(3, min(args.steps, 10))
    f_ms = reduce_max(statistics.median(timed_steps(fwd, n_it, flush)), world)
    fb_ms = reduce_max(statistics.median(timed_steps(fwd_bwd, n_it, flush)), world)
    fl_fb = flops(cfg)
    peak_tf = float(peaks.get("bf16_tflops", 1590.0))
    return {"config": "B_d1", "split": f"axis 0 (L={cfg.extent[0]}) over {world} ranks",
            "halo_rows": cp.split.halo, "slab_rows_rank0": list(cp.split.slab(0)),
            "recompute_overhead": round((e0 - s0) / (b - a) - 1.0, 4),
            "fwd_ms": round(f_ms, 4), "fwd_bwd_ms": round(fb_ms, 4),
            "fwd_bwd_tflops": round(fl_fb / (fb_ms * 1e-3) / 1e12, 3),
            "fwd_bwd_tensor_peak_frac": round(fl_fb / (fb_ms * 1e-3) / 1e12 / (world * peak_tf), 5)}


def run_native(args, world, rank, local):
    na_peaks, peak_src = load_peaks()
    R = Runner(rank, world)
    cfg0 = R.cfgs[0]
    step_flops = sum(flops(c) for c in R.cfgs)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > L2 (126 MB)

    for _ in range(args.warmup):
        R.step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    barrier(world)
    torch.cuda.synchronize()
    per_step = timed_steps(R.step, args.steps, flush)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    launches_per_step = R.launches
    ms_rank = sum(per_step) / args.steps
    ms = reduce_max(ms_rank, world)
    value = step_flops / (ms * 1e-3) / 1e12  # whole config over all ranks (strong split)

    # fwd-only timing (for the "fwd ms" half of the metric)
    fwd_ms = reduce_max(sum(timed_steps(R.fwd_only, max(2, args.steps // 2), flush)) /
                        max(2, args.steps // 2), world)

    # per-kernel device times, live, via the library's event hook on the launch stream
    R.na.profile_enable(True)
    prof_steps = 2
    for _ in range(prof_steps):
        flush.zero_()
        R.step()
    rec = R.na.profile_collect()
    R.na.profile_enable(False)
    per_kernel = {}
    for name, t in rec:
        d = per_kernel.setdefault(name, [0.0, 0])
        d[0] += t
        d[1] += 1
    dominant = max(per_kernel, key=lambda n: per_kernel[n][0])
    dom_ms, dom_n = per_kernel[dominant]
    avg_launch_ms = dom_ms / dom_n
    n_local = R.bh[1] - R.bh[0]  # this rank's slices per launch
    alg_bytes = algorithmic_bytes(cfg0, dominant, n_local)
    achieved = alg_bytes / (avg_launch_ms * 1e-3) / 1e9
    peak = float(na_peaks["hbm_gbs"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dominant)
        except Exception:
            traffic = None
    shares = {n: round(v[0] / sum(x[0] for x in per_kernel.values()), 4) for n, v in per_kernel.items()}
    # every kernel of the step against the HBM roofline (algorithmic bytes of
    # config B_d1 per launch / average launch time)
    per_kernel_roof = {}
    for n, (tot, cnt) in per_kernel.items():
        ms_avg = tot / cnt
        key = "fna_bwd_pre" if n.startswith("fna_bwd_pre") else n
        try:
            gbs = algorithmic_bytes(cfg0, key, n_local) / (ms_avg * 1e-3) / 1e9
        except KeyError:
            continue
        per_kernel_roof[n] = {"avg_launch_ms": round(ms_avg, 5), "achieved_gbs": round(gbs, 1),
                              "hbm_frac": round(gbs / peak, 4)}

    # end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        host = [t.cpu().pin_memory() for t in (R.q, R.k, R.v, R.do)]
        dev = [torch.empty_like(t) for t in (R.q, R.k, R.v, R.do)]
        outs_host = [[torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                      for t in (o, lse, *g)] for (o, lse, g, _) in R.outs]

        # Pipelined over chunks of (b,h) slices on three streams: chunk c's
        # inputs go host -> device on one copy stream while chunk c-1 computes
        # (every variant, fwd + bwd, through the public API on slice views)
        # and chunk c-2's outputs go device -> host on the other (PCIe is
        # full duplex); the step ends when the last output has landed.
        n_loc = R.bh[1] - R.bh[0]
        n_chunks = min(8, n_loc)
        bounds = [(n_loc * i // n_chunks, n_loc * (i + 1) // n_chunks) for i in range(n_chunks)]
        s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()

        def e2e_step():
            comp = torch.cuda.current_stream()
            s_h2d.wait_stream(comp)  # nothing starts before the step's start event
            for a, b in bounds:
                with torch.cuda.stream(s_h2d):
                    for h, d in zip(host, dev):
                        d[:, a:b].copy_(h[:, a:b], non_blocking=True)
                comp.wait_stream(s_h2d)
                R.step(*(d[:, a:b] for d in dev), sl=(a, b))
                s_d2h.wait_stream(comp)
                with torch.cuda.stream(s_d2h):
                    for (o, lse, g, _), hs in zip(R.outs, outs_host):
                        for src, dst in zip((o, lse, *g), hs):
                            dst[:, a:b].copy_(src[:, a:b], non_blocking=True)
            comp.wait_stream(s_d2h)

        e2e_step()
        torch.cuda.synchronize()
        n_e2e = max(2, min(args.steps, 5))
        barrier(world)
        e_ms = reduce_max(sum(timed_steps(e2e_step, n_e2e)) / n_e2e, world)
        h2d = sum(t.numel() * t.element_size() for t in host)
        d2h = sum(t.numel() * t.element_size() for hs in outs_host for t in hs)
        e2e = {"value": step_flops / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "pipeline": f"{n_chunks} chunks of (b,h) slices: H2D / na_fwd+na_bwd / D2H on three "
                           "streams, pinned host buffers"}

    per_config = None
    if not args.no_per_config:
        per_config = per_config_table(args, world, rank, na_peaks)

    cp_res = None
    if world > 1 and not args.no_per_config:
        try:  # optional report item: never lose the bench line over it
            cp_res = cp_table(args, world, rank, na_peaks)
        except Exception as ex:  # pragma: no cover
            cp_res = {"error": f"{type(ex).__name__}: {ex}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample()
        except Exception as ex:  # pragma: no cover
            cpu = {"error": str(ex)}

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic unit-normal Q,K,V,dO (seeded per (b,h)); no weights",
        "config": {"workload": WORKLOAD, "variants": VARIANTS, "batch": cfg0.batch,
                   "heads": cfg0.heads, "seq_len": cfg0.tokens, "head_dim": cfg0.head_dim,
                   "kernel_size": 255,
                   "parallelism": f"B*H split over {world} GPU(s): rank g owns slices "
                                  f"[g*{cfg0.batch * cfg0.heads}/{world}, (g+1)*{cfg0.batch * cfg0.heads}/{world})",
                   "l2": "inputs 1.07 GB/step > 126 MB L2, plus a 256 MB L2 flush between steps "
                         "outside the timed events"},
        "fwd_ms_per_step": round(fwd_ms, 4),
        "tensor_peak_frac": round(value / world / float(na_peaks.get("bf16_tflops", 1590.0)), 4),
        "roofline": {"kernel": dominant, "bound": "hbm", "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "algorithmic_bytes_per_launch": alg_bytes,
                     "avg_launch_ms": round(avg_launch_ms, 5), "peak_source": peak_src,
                     "step_share": shares, "kernels": per_kernel_roof},
        "per_config": per_config,
        "context_parallel": cp_res,
        "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "env": env_info(),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ reference arm

def run_reference(args, world, rank):
    if rank != 0:
        return
    import oracle
    cores = oracle.num_threads()
    step, fl, desc = oracle_sample(1024, cores)
    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    sec = sum(ts) / len(ts)
    value = fl / sec / 1e12
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "sample": desc},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true",
                    help="skip the fwd / fwd+bwd table of every BASELINE.json config")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the per-config whole-slice oracle parity (and oracle timing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = init_dist()
    run_native(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
