"""Benchmark: the paper's "total bandwidth" (minimum bytes / runtime) of the
bucketed approximate top-k hot path on B200, plus rows/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1]
    python bench.py --impl reference ...      # the CPU reference arm

Default workload (north-star target, BASELINE.json configs[0]):
fp32, m=128 rows per GPU, n=65536, k=64, b=64, k_b=1, interleaved.
Under torchrun every rank selects its own 128-row batch (weak scaling, no
collective on the data path); the step time is the max over ranks.

One JSON line on rank 0.  `value` = whole-job GB/s with inputs resident in
HBM (K launches replayed from a CUDA graph over rotating input buffers
whose total exceeds 4x the 126 MB L2, so every launch reads cold HBM);
`e2e` = the same metric through the public API `approx_topk()` with pinned
host input, H2D + kernels + D2H of (values, indices) inside the timed
region; `roofline` = the fused kernel's achieved GB/s against the measured
HBM copy peak (MEASURED_PEAKS.json); `cpu_baseline` = the oracle port of
the reference algorithm (NumPy, all host cores) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# name: (dtype, m, n, k, b, kb, scaling, description)
CONFIGS = {
    "cfg1": ("f32", 128, 65536, 64, 64, 1, "weak",
             "cfg1: fp32 m=128 n=65536 k=64 b=64 k_b=1 interleaved (no stage 2)"),
    "cfg2_kb2": ("f32", 128, 65536, 16384, 8192, 2, "weak", "cfg2: fp32 m=128 n=65536 k=16384 b=8192 k_b=2"),
    "cfg2_kb4": ("f32", 128, 65536, 16384, 4096, 4, "weak", "cfg2: fp32 m=128 n=65536 k=16384 b=4096 k_b=4"),
    "cfg2_kb8": ("f32", 128, 65536, 16384, 2048, 8, "weak", "cfg2: fp32 m=128 n=65536 k=16384 b=2048 k_b=8"),
    "cfg3_r1": ("bf16", 128, 1 << 20, 256, 256, 1, "weak", "cfg3: bf16 m=128 n=2^20 k=256 b=256 k_b=1"),
    "cfg3_r2": ("bf16", 128, 1 << 20, 256, 512, 1, "weak", "cfg3: bf16 m=128 n=2^20 k=256 b=512 k_b=1"),
    "cfg3_r4": ("bf16", 128, 1 << 20, 256, 1024, 1, "weak", "cfg3: bf16 m=128 n=2^20 k=256 b=1024 k_b=1"),
    "cfg3_r8": ("bf16", 128, 1 << 20, 256, 2048, 1, "weak", "cfg3: bf16 m=128 n=2^20 k=256 b=2048 k_b=1"),
    "cfg4": ("bf16", 4096, 32768, 512, 512, 1, "weak", "cfg4: bf16 m=4096 n=32768 k=512 b=512 k_b=1"),
    "cfg5": ("bf16", 8192, 1 << 20, 65536, 65536, 2, "strong",
             "cfg5: bf16 m=8192 n=2^20 k=65536 b=65536 k_b=2 (ratio 2), rows sharded over GPUs"),
}
L2_BYTES = 126 * 2**20
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg1", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-context", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def min_bytes(m, n, k, vb):
    # reference bench.py:154: one input read + k (value, int64 index) writes per row
    return m * (n * vb + k * (vb + 8))


def measured_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg)
    except Exception:
        return None


# --------------------------------------------------------------------------- CPU arms
def cpu_sample(cfg, budget_s=12.0, max_iters=50):
    """Oracle port of the reference (NumPy, all host threads) on a bounded
    sample of the workload: whole batches for small configs, a row subset
    for the big ones.  Returns (GB/s, rows/s, cores, sample description)."""
    import numpy as np

    from oracle import bucketed_oracle as O

    dt, m, n, k, b, kb, _, _ = CONFIGS[cfg]
    vb = 4 if dt == "f32" else 2
    cores = os.cpu_count() or 1
    rows = m
    per_row = n * vb
    if rows * per_row > 64 * 2**20:  # bound memory/time: a row subset
        rows = max(1, min(m, (64 * 2**20) // per_row))
    rng = np.random.default_rng(0)
    x = rng.standard_normal((rows, n), dtype=np.float32)
    if dt == "bf16":
        u = x.view(np.uint32).astype(np.uint64)
        x = (((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32) << 16).view(np.float32)
    O.approx_topk(x, k, b, kb, workers=cores)  # warm
    times = []
    t_start = time.perf_counter()
    while len(times) < 3 or (time.perf_counter() - t_start < budget_s and len(times) < max_iters):
        t0 = time.perf_counter()
        O.approx_topk(x, k, b, kb, workers=cores)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > 4 * budget_s:
            break
    mean = statistics.mean(times)
    gbs = min_bytes(rows, n, k, vb) / mean / 1e9
    sample = (f"{len(times)} x approx_topk over {rows} of {m} rows (n={n}) with workers={cores}, "
              f"numpy oracle port, mean {mean*1e3:.1f} ms")
    return gbs, rows / mean, cores, sample


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    dt, m, n, k, b, kb, scaling, desc = CONFIGS[cfg]
    gbs, rows_s, cores, sample = cpu_sample(cfg, budget_s=max(5.0, 0.5 * args.steps / 10))
    vb = 4 if dt == "f32" else 2
    ms = min_bytes(m, n, k, vb) / (gbs * 1e9) * 1e3
    line = {
        "impl": "reference",
        "metric": "total bandwidth GB/s (min bytes/runtime)",
        "value": round(gbs, 4), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32" if dt == "f32" else dt,
        "data": "synthetic N(0,1)",
        "config": {"workload": desc, "rows_per_s": round(rows_s, 2)},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self.names = {
            0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
            0x0000000000000020: "sw_thermal_slowdown", 0x0000000000000040: "hw_thermal_slowdown",
            0x0000000000000080: "hw_power_brake_slowdown", 0x0000000000000001: "gpu_idle",
            0x0000000000000002: "applications_clocks_setting",
        }

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.names.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch

    import paper_2412_04358_b200 as btk
    from paper_2412_04358_b200.shard import local_rows

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    cfg = args.config
    dt, m_cfg, n, k, b, kb, scaling, desc = CONFIGS[cfg]
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dt]
    vb = 4 if dt == "f32" else 2
    if scaling == "weak":
        m_local, m_total = m_cfg, m_cfg * world
    else:
        sl = local_rows(m_cfg, world, rank)
        m_local, m_total = sl.stop - sl.start, m_cfg
    scheme = btk.BucketScheme(b, kb, btk.Assignment.INTERLEAVED)
    batch_bytes = m_local * n * vb
    nbuf = max(2, min(64, -(-4 * L2_BYTES // max(batch_bytes, 1))))
    free = torch.cuda.mem_get_info(dev)[0]
    while nbuf > 2 and nbuf * batch_bytes > 0.5 * free:
        nbuf -= 1
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    bufs = []
    for _ in range(nbuf):
        bufs.append(torch.randn((m_local, n), generator=gen, device=dev, dtype=torch.float32).to(tdt))
    op = btk.ApproxTopK(m_local, n, k, scheme, dtype=tdt, device=dev)
    launches_per_step = op.lib.btk_launch_count(m_local, n, k, b, kb, op.dt, op.layout, n)
    stream = torch.cuda.Stream(device=dev)
    K, W = args.steps, max(3, args.warmup)

    with torch.cuda.stream(stream):
        for i in range(W):
            op.launch(bufs[i % nbuf])
        torch.cuda.synchronize(dev)
        # capture K steps (rotating buffers) into one CUDA graph
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(K):
                op.launch(bufs[i % nbuf])
        graph.replay()
        torch.cuda.synchronize(dev)

        clocks = ClockSampler(local)
        with clocks:
            # keep the GPU loaded ~0.3 s so the sampler sees clocks under load
            t_end = time.perf_counter() + 0.3
            while time.perf_counter() < t_end:
                graph.replay()
                torch.cuda.synchronize(dev)
            barrier()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            barrier()
        ms_total = e0.elapsed_time(e1)
        # eager launches (host-launched, no graph) for reference
        torch.cuda.synchronize(dev)
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        for i in range(K):
            op.launch(bufs[i % nbuf])
        e3.record(stream)
        torch.cuda.synchronize(dev)
        ms_eager = e2.elapsed_time(e3) / K

    ms_step = max_over_ranks(ms_total / K)
    total_bytes = min_bytes(m_total, n, k, vb)
    value = total_bytes / (ms_step * 1e-3) / 1e9
    local_bytes = min_bytes(m_local, n, k, vb)
    achieved = local_bytes / ((ms_total / K) * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # correctness spot-check of the timed configuration (oracle = checker only)
    op.check_finite()

    # ---- e2e through the public API (pinned host in, host out)
    e2e = None
    if not args.no_e2e:
        host = bufs[0].cpu().pin_memory()
        hv = torch.empty((m_local, k), dtype=tdt).pin_memory()
        hi = torch.empty((m_local, k), dtype=torch.int64).pin_memory()
        for _ in range(2):
            r = btk.approx_topk(host, k, scheme)
            hv.copy_(r.values)
            hi.copy_(r.indices)
        torch.cuda.synchronize(dev)
        barrier()
        E = args.e2e_steps
        cur = torch.cuda.current_stream(dev)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(cur)
        for _ in range(E):
            r = btk.approx_topk(host, k, scheme)  # H2D + kernels + finite check
            hv.copy_(r.values)                     # D2H of the result
            hi.copy_(r.indices)
        s1.record(cur)
        torch.cuda.synchronize(dev)
        e2e_ms = max_over_ranks(s0.elapsed_time(s1) / E)
        e2e = {"value": round(total_bytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "ms_per_step": round(e2e_ms, 4),
               "h2d_bytes_per_step": int(m_local * n * vb),
               "d2h_bytes_per_step": int(m_local * k * (vb + 8)),
               "path": "paper_2412_04358_b200.approx_topk(pinned host tensor) + .copy_ to pinned host"}

    # ---- context: torch.topk and bucketed argmax on the same buffers
    context = None
    if not args.no_context:
        def time_fn(fn, iters=20):
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            z = torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(iters):
                fn(bufs[i % nbuf])
            z.record()
            torch.cuda.synchronize(dev)
            return a.elapsed_time(z) / iters
        t_topk = time_fn(lambda x: torch.topk(x, k, dim=-1, sorted=True))
        context = {"torch_topk_GBps": round(local_bytes / (t_topk * 1e-3) / 1e9, 2),
                   "torch_topk_ms": round(t_topk, 4)}
        if kb == 1 and b * kb == k and n % b == 0:
            t_am = time_fn(lambda x: x.view(m_local, n // b, b).argmax(1))
            context["bucketed_argmax_GBps"] = round(local_bytes / (t_am * 1e-3) / 1e9, 2)
        context["eager_ms_per_step"] = round(ms_eager, 4)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gbs, rows_s, cores, sample = cpu_sample(cfg)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": sample, "rows_per_s": round(rows_s, 2)}

    if rank == 0:
        line = {
            "metric": "total bandwidth GB/s (min bytes/runtime)",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": dt, "data": "synthetic N(0,1) (torch Philox on device)",
            "config": {"workload": desc, "rows_per_gpu": m_local, "rows_total": m_total, "n": n,
                       "k": k, "b": b, "k_b": kb, "assignment": "interleaved",
                       "rows_per_s": round(m_total / (ms_step * 1e-3), 1),
                       "l2": f"{nbuf} rotating input buffers = {nbuf * batch_bytes / 2**20:.0f} MiB "
                             f"(> L2 {L2_BYTES // 2**20} MiB): inputs larger than L2",
                       "timing": "K launches captured in one CUDA graph, CUDA events on the "
                                 "launch stream, max over ranks",
                       "path": "fused" if op.fused else "generic"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": ncu_traffic(cfg), "peak_source": peak_src,
                         "bytes_per_launch": local_bytes},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(K * launches_per_step),
            "clocks": clocks.summary(),
            "context": context,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
