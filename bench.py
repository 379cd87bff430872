"""Benchmark of the PCCL collective data plane on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload auto|hash|allreduce|quant|local]
                    [--impl ours|reference]

Workloads (BASELINE.json metric "All-reduce bus GB/s (1 GiB fp32, 2/4/8 B200);
quant/hash kernel HBM GB/s"):

* ``hash`` (default at N=1; config 4): simplehash of an 8.03 B-parameter bf16
  shared state laid out like Llama-3-8B (291 entries, 16.06 GB per GPU), one
  multi-entry launch per step; value = HBM GB/s (bytes hashed / time). At N>1
  every GPU hashes its own replica (replicas only: sync_shared_state hashes
  each peer's copy) and value is the aggregate.
* ``allreduce`` (default at N>1; config 2): in-place AVG all-reduce of 1 GiB
  fp32 per GPU over NVLink, W = N ring positions; value = bus GB/s
  (algbw * 2(W-1)/W, algbw = 1 GiB / max-over-ranks time).
* ``quant`` (config 3): u8-quantized AVG all-reduce of 1.2 B fp32 per GPU.
* ``local``: W=8 logical peers of 1 GiB each on one GPU (the reference's
  in-process RingSession shape); value = bus GB/s.

Inputs are synthetic (torch RNG) and larger than L2 (126 MB), so no L2 flush
is needed between steps. Timing: CUDA events on the launching stream, W >= 3
warm-up steps, barrier + synchronize around the timed region, max over ranks.
``--impl reference`` times the reference algorithm on host cores: the faster of
the oracle port (C simplehash on every host thread; the NumPy ring) and the
unmodified reference itself from ``baseline/_ref`` (its own simplehash, and
its own TCP ring through ``churncomm.cli bench``), both reported.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "All-reduce bus GB/s (1 GiB fp32, 2/4/8 B200); quant/hash kernel HBM GB/s"


def llama3_8b_layout() -> list[tuple[str, int]]:
    """(name, elements) of a Llama-3-8B-like state: 291 entries, 8.03 B params."""
    d, kv, ff, vocab, layers = 4096, 1024, 14336, 128256, 32
    out = [("embed", vocab * d)]
    for i in range(layers):
        out += [
            (f"l{i}.q", d * d), (f"l{i}.k", kv * d), (f"l{i}.v", kv * d), (f"l{i}.o", d * d),
            (f"l{i}.gate", ff * d), (f"l{i}.up", ff * d), (f"l{i}.down", d * ff),
            (f"l{i}.attn_norm", d), (f"l{i}.mlp_norm", d),
        ]
    out += [("norm", d), ("lm_head", vocab * d)]
    return out


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML during the timed
    region (a sample at start, every `period` s, and at stop)."""

    REASONS = {  # nvmlClocksEventReason* bits
        "sw_power_cap": 0x4,
        "hw_slowdown": 0x8,
        "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
    }

    def __init__(self, index: int, period: float = 0.1):
        """NVML is initialised here, before warm-up: on a fresh box nvmlInit
        takes long and holds driver locks, which stalled the first timed
        all-reduces of a run (2.5 -> 3.5-4.7 ms at W=4)."""
        self.index = index
        self.period = period
        self.samples = []
        self.stop_ev = threading.Event()
        self.thread = None
        self.h = None
        if os.environ.get("BENCH_NO_CLOCKS"):
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.samples.clear()
        except Exception:  # noqa: BLE001
            self.h = None

    def _sample(self):
        import pynvml

        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        try:
            bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except AttributeError:  # older bindings
            bits = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, bits))

    def start(self):
        if self.h is None:
            return
        self._sample()

        def loop():
            while not self.stop_ev.wait(self.period):
                self._sample()

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": ["nvml unavailable"]}
        self.stop_ev.set()
        self.thread.join(timeout=5)
        self._sample()
        sm = sorted(x for x, _ in self.samples)
        reasons = sorted({nm for _, b in self.samples for nm, bit in self.REASONS.items() if b & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "samples": len(sm), "reasons": reasons,
                "source": "NVML (nvidia_ml_py), sampled during the timed region"}


def ncu_traffic(key: str):
    """DRAM bytes per launch of the workload's dominant kernel from the committed
    ncu capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")) as f:
            e = json.load(f).get(key)
        return int(e["bytes"]) if e else None
    except (OSError, ValueError, KeyError):
        return None


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "src": "measured"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "src": "fallback"}


NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_init(n: int):
    import torch
    import torch.distributed as dist

    if n <= 1 and "RANK" not in os.environ:
        return 0, 1, 0
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(n)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available() and torch.cuda.device_count() > 0:
        local %= torch.cuda.device_count()  # >1 rank per GPU only when oversubscribed (W=8 dry run on 4 GPUs)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def bench_hash(args, rank, world, local):
    import torch

    from paper_2505_14065_b200.sharedstate import simplehash_many_async

    dev = torch.device("cuda", local)
    clocks = ClockSampler(local)  # NVML initialised before warm-up
    layout = llama3_8b_layout()
    total_elems = sum(n for _, n in layout)
    state = torch.empty(total_elems, dtype=torch.bfloat16, device=dev)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    # random bf16 bit patterns (fills all 16 GB quickly)
    state.view(torch.int16).random_(-32768, 32767, generator=g)
    views, off = [], 0
    for _, n in layout:
        views.append(state[off : off + n])
        off += n
    nbytes = total_elems * 2
    out = torch.empty(len(views), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        simplehash_many_async(views, out)
    torch.cuda.synchronize(dev)
    barrier(world)
    clocks.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        simplehash_many_async(views, out)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1) / args.steps
    clk = clocks.stop()
    barrier(world)
    ms_max = max_over_ranks(ms, world)
    # per step: the batch kernel, the big-entry kernel and the 1-CTA gate
    # kernel between them (replayed as one CUDA graph of the plan)
    launches = 3 * args.steps

    # the two 1.05 GB entries alone (the bitsliced big-entry kernel) and the
    # other 289 alone (the TMA batch kernel): how the concurrent launch overlaps
    def time_views(vs, reps=3):
        simplehash_many_async(vs, out[: len(vs)])
        t0.record(stream)
        for _ in range(reps):
            simplehash_many_async(vs, out[: len(vs)])
        t1.record(stream)
        torch.cuda.synchronize(dev)
        return t0.elapsed_time(t1) / reps

    big_ms = time_views([views[0], views[-1]])
    rest_ms = time_views(views[1:-1])

    # parity outside the timed region: every digest against the C oracle
    parity = None
    if not args.no_parity:
        from oracle import simplehash as osh

        simplehash_many_async(views, out)
        got = [int(x) & 0xFFFFFFFFFFFFFFFF for x in out.cpu().tolist()]
        host = state.view(torch.uint8).cpu().numpy()
        bufs, off = [], 0
        for _, n in layout:
            bufs.append(host[off : off + 2 * n])
            off += 2 * n
        order = sorted(range(len(bufs)), key=lambda i: -bufs[i].size)
        want = dict(zip(order, osh.simplehash_many_c([bufs[i] for i in order], threads=os.cpu_count() or 8)))
        bad = sum(got[i] != want[i] for i in range(len(bufs)))
        parity = {"status": "ok" if bad == 0 else "MISMATCH", "checked": f"{len(bufs) - bad}/{len(bufs)} digests "
                  "equal oracle/simplehash.c (all 291 entries, 16.06 GB)"}
        del host, bufs

    # e2e: host state (pinned) -> device, hash, digests -> host
    e2e = None
    if not args.no_e2e:
        host = torch.empty(total_elems, dtype=torch.bfloat16, pin_memory=True)
        host.copy_(state, non_blocking=False)
        digests = torch.empty(len(views), dtype=torch.int64, pin_memory=True)
        def e2e_step():
            state.copy_(host, non_blocking=True)
            simplehash_many_async(views, out)
            digests.copy_(out, non_blocking=True)
        e2e_step()
        torch.cuda.synchronize(dev)
        k = max(1, min(args.steps, 3))
        barrier(world)
        t0.record(stream)
        for _ in range(k):
            e2e_step()
        t1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = max_over_ranks(t0.elapsed_time(t1) / k, world)
        e2e = {"value": round(world * nbytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": len(views) * 8, "ms_per_step": round(e2e_ms, 3)}
        del host

    pk = peaks()
    achieved = nbytes / (ms * 1e-3) / 1e9
    result = {
        "value": round(world * nbytes / (ms_max * 1e-3) / 1e9, 2),
        "unit": "GB/s",
        "ms_per_step": round(ms_max, 4),
        "scaling": "weak",
        "dtype": "u8",
        "config": {"workload": "config4-hash: simplehash of Llama-3-8B-like bf16 shared state (291 entries, 16.06 GB/GPU), one multi-entry launch per step",
                   "entries": len(views), "bytes_per_gpu": nbytes, "largest_entry_bytes": views[0].numel() * 2,
                   "l2": "inputs 16 GB >> 126 MB L2; no flush needed", "replicas": world},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / pk["hbm_gbs"], 4),
                     "traffic": ncu_traffic("hash_config4"),
                     "peak_src": pk["src"],
                     "kernel": "simplehash_batch_kernel (289 entries, TMA ring) + simplehash_big_kernel "
                               "(the two 1.05 GB entries, bitsliced lo scan), one call, concurrent",
                     "algorithmic_bytes_per_launch": nbytes,
                     "big_entries_alone_ms": round(big_ms, 3),
                     "rest_alone_ms": round(rest_ms, 3),
                     "hbm_floor_ms": round(nbytes / (pk["hbm_gbs"] * 1e9) * 1e3, 3)},
        "parity": parity,
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_hash_baseline(layout)
    return result


def hash_sample(layout):
    """Bounded CPU sample of the config-4 workload: every 9th entry (largest
    first order keeps one 1.05 GB embedding), random bytes."""
    import numpy as np

    sel = [n for i, (_, n) in enumerate(layout) if i % 9 == 0]
    rng = np.random.default_rng(7)
    return [rng.integers(0, 256, 2 * n, dtype=np.uint8) for n in sel]


REF_PKG = os.path.join(ROOT, "baseline", "_ref")  # the unmodified reference, pip-installed by build()


def reference_own_hash(bufs, want=None, max_bytes=1200 << 20) -> dict | None:
    """The reference's own ``churncomm.sharedstate.simplehash`` (SURVEY 8(d)
    (iv)), timed beside the C port on part of the same sample: workers=1, its
    fastest setting (2 / 4 / 8 workers measured 0.28 / 0.14 / 0.07 GB/s against
    0.50). Reported only; the port stays the baseline value. ``want``: the
    port's digests of ``bufs``, compared with the reference's own."""
    if not os.path.isdir(os.path.join(REF_PKG, "churncomm")):
        return None
    sys.path.insert(0, REF_PKG)
    try:
        from churncomm import sharedstate as ref_ss
    except Exception as e:  # noqa: BLE001 - report, never fail the bench line
        return {"unavailable": f"{type(e).__name__}: {e}"[:160]}
    finally:
        sys.path.remove(REF_PKG)
    picked, nb = [], 0
    for i in sorted(range(len(bufs)), key=lambda i: bufs[i].size):
        if nb + bufs[i].size > max_bytes and picked:
            break
        picked.append(i)
        nb += bufs[i].size
    t = time.perf_counter()
    got = [ref_ss.simplehash(bufs[i], workers=1) for i in picked]
    dt = time.perf_counter() - t
    d = {"value": round(nb / dt / 1e9, 3), "unit": "GB/s", "cores": 1,
         "impl": "churncomm.sharedstate.simplehash(buffer, workers=1), unmodified reference (baseline/_ref)",
         "sample": f"{len(picked)} of the sample's entries ({nb / 1e6:.0f} MB)"}
    if want is not None:
        d["digests_equal_port"] = all(int(got[k]) == int(want[i]) for k, i in enumerate(picked))
    return d


def reference_own_ring(world: int, nbytes: int = 16 << 20) -> dict | None:
    """The reference's own CPU ring all-reduce through its own benchmark CLI
    (``python -m churncomm.cli bench``: a local master and
    one process per peer over TCP loopback), AVG of `nbytes` per peer, pool 2,
    3 repeats; busbw = algbw * 2(W-1)/W. Reported beside the port."""
    import subprocess

    if not os.path.isdir(os.path.join(REF_PKG, "churncomm")):
        return None
    w = max(world, 2)
    env = dict(os.environ, PYTHONPATH=REF_PKG, PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "churncomm.cli", "bench", "--world", str(w), "--bytes", str(nbytes),
           "--op", "avg", "--pool", "2", "--repeats", "3"]
    try:
        out = subprocess.run(cmd, env=env, cwd="/tmp", capture_output=True, text=True, timeout=180)
        rep = None
        for line in out.stdout.splitlines() + out.stderr.splitlines():
            if '"bench_report"' in line:
                rep = json.loads(line[line.index("{"):])
        if rep is None:
            return {"unavailable": f"no bench_report (exit {out.returncode})"}
    except Exception as e:  # noqa: BLE001 - report, never fail the bench line
        return {"unavailable": f"{type(e).__name__}: {e}"[:160]}
    algbw = rep["bytes_per_op"] / rep["time_s"] / 1e9
    return {"value": round(algbw * 2 * (w - 1) / w, 4), "unit": "GB/s", "cores": w,
            "ms_per_op": round(rep["time_s"] * 1e3, 2),
            "impl": "churncomm.cli bench (unmodified reference from baseline/_ref): TCP loopback ring, one process per peer",
            "sample": f"W={w}, {nbytes >> 20} MiB f32 per peer, AVG, pool 2, 3 repeats ({rep['time_s'] * 1e3:.1f} ms per op)"}


def cpu_hash_baseline(layout) -> dict:
    from oracle import simplehash as osh

    bufs = hash_sample(layout)
    threads = os.cpu_count() or 1
    nb = sum(b.size for b in bufs)
    t = time.perf_counter()
    want = osh.simplehash_many_c(bufs, threads=threads)
    dt = time.perf_counter() - t
    out = {"value": round(nb / dt / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "port",
           "sample": f"{len(bufs)} of 291 config-4 entries ({nb / 1e9:.2f} GB), oracle/simplehash.c on {threads} threads"}
    own = reference_own_hash(bufs, want)
    if own is not None:
        out["reference_own"] = own
    return out


def bench_allreduce(args, rank, world, local, quantize=False):
    import torch

    from paper_2505_14065_b200.ring_ipc import DeviceRing

    dev = torch.device("cuda", local)
    clocks = ClockSampler(local)  # NVML initialised before warm-up
    n = args.elems or ((1 << 28) if not quantize else 1_200_000_000)
    op = "avg"
    g = torch.Generator(device=dev).manual_seed(rank)
    src = torch.randn(n, generator=g, device=dev) * (1e-2 if quantize else 1.0)
    buf = torch.empty_like(src)
    esz = 4
    ring = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(n, world, esz, quantize))
    if not args.no_register:
        ring.register(buf)  # one-time collective setup: peers read buf in place (zero-copy)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        buf.copy_(src)
        ring.run_all_reduce(buf, op, quantize=quantize)
    torch.cuda.synchronize(dev)
    # K ops enqueued back to back (all_reduce_async), events around all K;
    # every op's result is awaited after the timed region. AVG of AVG keeps the
    # values bounded, so no re-seeding is needed between steps.
    buf.copy_(src)
    torch.cuda.synchronize(dev)
    barrier(world)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tickets = []
    for _ in range(args.steps):
        if len(tickets) >= 32:  # the engine keeps up to 64 attempts in flight
            ring.await_reduce(tickets.pop(0))
        tickets.append(ring.all_reduce_async(buf, op, quantize=quantize))
    e1.record(stream)
    for t in tickets:
        ring.await_reduce(t)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    barrier(world)
    ms_max = max_over_ranks(ms, world)
    S = n * esz
    algbw = S / (ms_max * 1e-3) / 1e9
    busbw = algbw * 2 * (world - 1) / world if world > 1 else 0.0
    # e2e: pinned host buffer -> device, all-reduce, result -> host
    e2e = None
    if not args.no_e2e:
        host_in = src.cpu().pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()
        k = max(1, min(args.steps, 3))
        barrier(world)
        e0.record(stream)
        for _ in range(k):
            buf.copy_(host_in, non_blocking=True)
            t = ring.all_reduce_async(buf, op, quantize=quantize)
            host_out.copy_(buf, non_blocking=True)
            ring.await_reduce(t)  # the step's result is on the host
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / k, world)
        e2e_alg = S / (e2e_ms * 1e-3) / 1e9
        e2e = {"value": round(e2e_alg * 2 * (world - 1) / world if world > 1 else e2e_alg, 2), "unit": "GB/s",
               "h2d_bytes_per_step": S, "d2h_bytes_per_step": S, "ms_per_step": round(e2e_ms, 3)}
    # parity outside the timed region: one fresh all-reduce of the seeded
    # inputs; every rank checks the chunk it owns against the oracle (peers'
    # inputs regenerated from their seeds on this device)
    parity = None
    if not args.no_parity:
        from oracle import ring as oring

        buf.copy_(src)
        ring.run_all_reduce(buf, op, quantize=quantize)
        torch.cuda.synchronize(dev)
        scale = 1e-2 if quantize else 1.0

        def peer_input(p):
            gp = torch.Generator(device=dev).manual_seed(p)
            return torch.randn(n, generator=gp, device=dev) * scale

        bounds = oring.chunk_bounds(n, world)
        c = (ring.position + 1) % world  # the chunk this position owns (folded last here)
        lo, hi = bounds[c]
        spans = [peer_input((c + k) % world)[lo:hi].cpu().numpy() for k in range(world)]
        if world > 1:
            want = oring.reduce_chunk(spans, oring.ReduceOp.AVG, quantize, world)
        else:  # W = 1: finalize only, never quantized (client.py:896-900)
            want = spans[0]
        ok = buf[lo:hi].cpu().numpy().tobytes() == want.tobytes()
        ok = max_over_ranks(0.0 if ok else 1.0, world) == 0.0
        parity = {"status": "ok" if ok else "MISMATCH",
                  "checked": f"the chunk each of the {world} ranks owns ({hi - lo} elements) "
                             "bit-equal to oracle.ring.reduce_chunk"}
    nvl_bytes = 2 * (world - 1) / world * S  # per-GPU NVLink ingress (plain)
    # plain: fold, push gather, 3 barriers; quantized (fused schedule): range,
    # barrier 0, W-1 step kernels, the fused adoption+gather kernel
    launches_per_op = (2 + 3) if not quantize else (1 + 1 + (world - 1) + 1)
    if not quantize:
        # NVLink-bound: per-GPU ingress 2(W-1)/W * S against the measured peer copy
        roof = {"bound": "nvlink", "achieved": round(nvl_bytes / (ms_max * 1e-3) / 1e9, 1),
                "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                "frac": round(nvl_bytes / (ms_max * 1e-3) / 1e9 / NVLINK_PEER_GBS, 4), "traffic": None,
                "peak_src": "measured peer copy 770 GB/s per direction (B200_PROFILING.md); "
                            "both-ways SM pull measured 655 (tools/micro/p2p_micro.cu)",
                "algorithmic_bytes_per_gpu": int(nvl_bytes)}
    else:
        # HBM-bound: per GPU (W-1) reduce steps of 14 B/elem of a chunk
        # (quantize 5 + dequant-accumulate 9), the owner's adoption 13 B, and the
        # gather's (W-1) x 5 B (codes in, floats out) = (19(W-1) + 13) * n_c bytes
        n_c = (n + world - 1) // world
        hbm_bytes = (19 * (world - 1) + 13) * n_c
        pk = peaks()
        ach = hbm_bytes / (ms_max * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / pk["hbm_gbs"], 4), "traffic": None, "peak_src": pk["src"],
                "traffic_step_kernel": (ncu_traffic("quant_w2_1200M_step") if world == 2 and n == 1_200_000_000 else None),
                "algorithmic_bytes_per_gpu": hbm_bytes,
                "nvlink_bytes_per_gpu": 2 * (world - 1) * n_c}
        # the schedule's own HBM traffic, incl. the backup the reference keeps
        # (collective.py:501-504) and the codes peers push into this GPU, per
        # n_c: range+backup 8; per step 14 (quantize 4, codes in 1, backup +
        # range 4+1+4) plus 1 from step 2 on (the previous step's codes: the
        # running partial is recomputed, never stored); adoption 9 (x, codes,
        # write-back); gather (W-1) x 6 (codes in + read, floats out)
        full = (8 + 14 * (world - 1) + max(world - 2, 0) + 9 + 6 * (world - 1)) * n_c
        roof["schedule_bytes_per_gpu"] = full
        roof["frac_of_schedule_floor"] = round(full / (ms_max * 1e-3) / 1e9 / pk["hbm_gbs"], 4)
    result = {
        "value": round(busbw, 2),
        "unit": "GB/s",
        "ms_per_step": round(ms_max, 4),
        "scaling": "weak",
        "dtype": "f32",
        "config": {"workload": f"config{'3' if quantize else '2'}: in-place AVG all-reduce{' u8-quantized' if quantize else ''} of {S / 2**30:.3f} GiB fp32 per GPU over NVLink, W={world}",
                   "elements_per_gpu": n, "ring": list(range(world)), "algbw_GBps": round(algbw, 2),
                   "buffer": "unregistered (staged copy-in)" if args.no_register else "registered once (DeviceRing.register, zero-copy reads)",
                   "busbw_definition": "algbw*2(W-1)/W", "l2": "1 GiB inputs > 126 MB L2"},
        "roofline": roof,
        "parity": parity,
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches_per_op * args.steps,
    }
    ring.close()
    return result


def bench_sweep(args, rank, world, local):
    """Config 2's bandwidth sweep: in-place AVG all-reduce of S = 1 MiB .. 4 GiB
    fp32 per GPU (x4 steps), K ops back to back per size (CUDA events, max over
    ranks), registered buffer. value = busbw at 1 GiB."""
    import torch

    from paper_2505_14065_b200.ring_ipc import DeviceRing

    dev = torch.device("cuda", local)
    clocks = ClockSampler(local)  # NVML initialised before warm-up
    sizes = [1 << e for e in range(20, 33, 2)]  # bytes: 1 MiB, 4 MiB, ..., 4 GiB
    nmax = sizes[-1] // 4
    g = torch.Generator(device=dev).manual_seed(rank)
    src = torch.randn(nmax, generator=g, device=dev)
    buf = torch.empty_like(src)
    ring = DeviceRing(device=dev, capacity_bytes=DeviceRing.required_bytes(nmax, world, 4, False))
    ring.register(buf)
    stream = torch.cuda.current_stream(dev)
    rows = []
    clocks.start()
    for S in sizes:
        n = S // 4
        view = buf[:n]
        view.copy_(src[:n])
        steps = max(5, min(200, (64 << 20) // S * 5))
        for _ in range(max(3, args.warmup)):
            ring.run_all_reduce(view, "avg")
        torch.cuda.synchronize(dev)
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tickets = []
        for _ in range(steps):
            if len(tickets) >= 32:
                ring.await_reduce(tickets.pop(0))
            tickets.append(ring.all_reduce_async(view, "avg"))
        e1.record(stream)
        for t in tickets:
            ring.await_reduce(t)
        torch.cuda.synchronize(dev)
        ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
        algbw = S / (ms * 1e-3) / 1e9
        busbw = algbw * 2 * (world - 1) / world if world > 1 else 0.0
        rows.append({"bytes": S, "us_per_op": round(ms * 1e3, 2), "algbw_GBps": round(algbw, 1),
                     "busbw_GBps": round(busbw, 1), "frac_of_770": round(busbw / NVLINK_PEER_GBS, 4),
                     "frac_of_900": round(busbw / 900.0, 4), "ops": steps})
    clk = clocks.stop()
    ring.close()
    at1g = next(r for r in rows if r["bytes"] == 1 << 30)
    return {
        "value": at1g["busbw_GBps"], "unit": "GB/s", "ms_per_step": round(at1g["us_per_op"] / 1e3, 4),
        "scaling": "weak", "dtype": "f32",
        "config": {"workload": f"config2 sweep: AVG all-reduce of 1 MiB..4 GiB fp32 per GPU, W={world}, registered buffer",
                   "busbw_definition": "algbw*2(W-1)/W", "sweep": rows},
        "roofline": {"bound": "nvlink", "achieved": round(at1g["busbw_GBps"], 1), "peak": NVLINK_PEER_GBS,
                     "unit": "GB/s", "frac": at1g["frac_of_770"], "traffic": None,
                     "peak_src": "measured peer copy 770 GB/s per direction (B200_PROFILING.md); nominal 900"},
        "clocks": clk, "e2e": None, "gpu_launches": None,
    }


def bench_local(args, rank, world, local):
    import torch

    from paper_2505_14065_b200 import LocalRing

    dev = torch.device("cuda", local)
    clocks = ClockSampler(local)  # NVML initialised before warm-up
    w = 8
    n = args.elems or (1 << 28)
    g = torch.Generator(device=dev).manual_seed(0)
    srcs = [torch.randn(n, generator=g, device=dev) for _ in range(w)]
    bufs = [torch.empty_like(s) for s in srcs]
    ring = LocalRing(w, device=dev, backup=False)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        ring.launch(bufs, "avg")
    torch.cuda.synchronize(dev)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ring.launch(bufs, "avg")
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    S = n * 4
    busbw = S / (ms * 1e-3) / 1e9 * 2 * (w - 1) / w
    hbm = 2 * w * S / (ms * 1e-3) / 1e9  # W reads + W writes per element
    pk = peaks()
    return {
        "value": round(busbw, 2), "unit": "GB/s", "ms_per_step": round(ms, 4), "scaling": "weak", "dtype": "f32",
        "config": {"workload": "8 logical ring peers x 1 GiB fp32 on one GPU, AVG (RingSession shape)", "elements_per_peer": n},
        "roofline": {"bound": "hbm", "achieved": round(hbm, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": round(hbm / pk["hbm_gbs"], 4),
                     "traffic": ncu_traffic("local_w8_1GiB") if n == 1 << 28 and w == 8 else None,
                     "kernel": "local_fold_all_kernel"},
        "clocks": clk, "e2e": None, "gpu_launches": args.steps,
    }


def bench_async(args, rank, world, local):
    """Config 5 shape without the fault: two u8-quantized AVG all-reduces (tags 0
    and 1, two halves of a pseudo-gradient) in flight together through the
    Communicator API (client.py:802-847: one engine + stream per pool slot).
    A step enqueues both and awaits both on the host."""
    import torch

    from paper_2505_14065_b200.communicator import Communicator
    from paper_2505_14065_b200.ring_ipc import DeviceRing

    dev = torch.device("cuda", local)
    clocks = ClockSampler(local)  # NVML initialised before warm-up
    torch.cuda.set_device(dev)
    n = args.elems or 600_000_000
    g = torch.Generator(device=dev).manual_seed(rank)
    src = [torch.randn(n, generator=g, device=dev) * 1e-2 for _ in range(2)]
    bufs = [s.clone() for s in src]
    comm = Communicator(device=dev, pool_size=2, capacity_bytes=DeviceRing.required_bytes(n, world, 4, True))

    def step():
        hs = [comm.all_reduce_async(bufs[t], t, "avg", quantize=True) for t in range(2)]
        for h in hs:
            r = comm.await_async_reduce(h)
            if not r.completed:
                raise RuntimeError(f"async all-reduce aborted: {r.reason}")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    barrier(world)
    clocks.start()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    for st in comm.streams:
        stream.wait_stream(st)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    S = 2 * n * 4
    algbw = S / (ms * 1e-3) / 1e9
    busbw = algbw * 2 * (world - 1) / world if world > 1 else 0.0
    n_c = (n + world - 1) // world
    # the fused schedule's HBM traffic, both tags (per-n_c terms as in bench_allreduce)
    full = 2 * (8 + 14 * (world - 1) + max(world - 2, 0) + 9 + 6 * (world - 1)) * n_c
    pk = peaks()
    comm.close()
    return {
        "value": round(busbw, 2), "unit": "GB/s", "ms_per_step": round(ms, 4), "scaling": "weak", "dtype": "f32",
        "config": {"workload": f"config5 (no fault): two concurrent u8-quantized AVG all-reduces of {n} fp32 each "
                               f"per GPU (tags 0/1, Communicator pool of 2), W={world}",
                   "elements_per_gpu_per_tag": n, "algbw_GBps": round(algbw, 2), "busbw_definition": "algbw*2(W-1)/W",
                   "timing": "host enqueue + await of both tags inside the timed region"},
        "roofline": {"bound": "hbm", "achieved": round(full / (ms * 1e-3) / 1e9, 1), "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": round(full / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], 4), "traffic": None,
                     "peak_src": pk["src"], "schedule_bytes_per_gpu": full},
        "clocks": clk, "e2e": None, "gpu_launches": 2 * (world + 2) * args.steps,
    }


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm on host cores (port and the reference itself)
# ---------------------------------------------------------------------------
def reference_arm(args, workload, world):
    import numpy as np

    if workload == "hash":
        layout = llama3_8b_layout()
        bufs = hash_sample(layout)
        from oracle import simplehash as osh

        threads = os.cpu_count() or 1
        nb = sum(b.size for b in bufs)
        for _ in range(min(args.warmup, 1)):
            osh.simplehash_many_c(bufs[-4:], threads=threads)
        t = time.perf_counter()
        steps = max(1, min(args.steps, 2))
        for _ in range(steps):
            want = osh.simplehash_many_c(bufs, threads=threads)
        dt = (time.perf_counter() - t) / steps
        v = round(world * nb / dt / 1e9, 3)
        cpu = {"value": v, "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"{len(bufs)} of 291 entries ({nb / 1e9:.2f} GB) via oracle/simplehash.c"}
        own = reference_own_hash(bufs, want)
        if own is not None:
            cpu["reference_own"] = own
        return {"metric": METRIC, "value": v, "unit": "GB/s", "impl": "reference", "n_gpus": world,
                "steps": steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": {"workload": "config4-hash (bounded sample)"},
                "cpu_baseline": cpu,
                "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    from oracle import ring as oring

    w = max(world, 2)
    n = 1 << 22  # bounded sample: 16 MiB per rank
    rng = np.random.default_rng(0)
    bufs = [rng.normal(0, 1, n).astype(np.float32) for _ in range(w)]
    quant = workload in ("quant", "async")
    oring.ring_allreduce(bufs, oring.ReduceOp.AVG, quantize=quant)
    steps = max(1, min(args.steps, 3))
    t = time.perf_counter()
    for _ in range(steps):
        oring.ring_allreduce(bufs, oring.ReduceOp.AVG, quantize=quant)
    dt = (time.perf_counter() - t) / steps
    algbw = n * 4 / dt / 1e9
    v = round(algbw * 2 * (w - 1) / w, 4)
    cpu = {"value": v, "unit": "GB/s", "cores": 1, "kind": "port",
           "sample": f"oracle.ring.ring_allreduce W={w}, 4 Mi f32 per rank, AVG{' u8' if quant else ''}"}
    ms = dt * 1e3
    if not quant:  # the reference's bench CLI has no quantize flag (cli.py:59-70)
        own = reference_own_ring(w)
        if own is not None and "value" in own and own["value"] > v:
            # the reference's own ring (one process per peer) beats the
            # single-process port: the arm reports the faster of the two
            cpu = {"value": own["value"], "unit": "GB/s", "cores": own["cores"], "kind": "reference",
                   "sample": f"{own['sample']}; {own['impl']}", "port": cpu}
            v, ms = own["value"], own["ms_per_op"]
        elif own is not None:
            cpu["reference_own"] = own
    return {"metric": METRIC, "value": v, "unit": "GB/s", "impl": "reference", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{workload} W={w} (bounded sample 16 MiB/rank)"},
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="auto", choices=["auto", "hash", "allreduce", "quant", "async", "local", "sweep"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--elems", type=int, default=0, help="override elements per GPU (allreduce/quant/local)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check after the timed region")
    ap.add_argument("--no-register", action="store_true", help="all-reduce: stage through the workspace instead of registering the buffer")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world_env = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    workload = args.workload
    if workload == "auto":
        workload = "hash" if world_env <= 1 else "allreduce"

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        print(json.dumps(reference_arm(args, workload, world_env)))
        return

    rank, world, local = dist_init(args.gpus)
    if workload == "hash":
        res = bench_hash(args, rank, world, local)
    elif workload == "allreduce":
        res = bench_allreduce(args, rank, world, local, quantize=False)
    elif workload == "quant":
        res = bench_allreduce(args, rank, world, local, quantize=True)
    elif workload == "async":
        res = bench_async(args, rank, world, local)
    elif workload == "sweep":
        res = bench_sweep(args, rank, world, local)
    else:
        res = bench_local(args, rank, world, local)
    line = {"metric": METRIC, "value": res.pop("value"), "unit": res.pop("unit"), "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res.pop("ms_per_step"),
            "higher_is_better": True, "scaling": res.pop("scaling"), "vs_baseline": None,
            "dtype": res.pop("dtype"), "data": "synthetic"}
    line.update(res)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
