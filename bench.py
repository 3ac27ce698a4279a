"""Benchmark of the LRAMM approximate-GEMM hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

One step = one approximate GEMM D ~= A.B through the whole pipeline (randomised SVD of
both operands with quantised int8 / packed-int4 sketch, power and projection GEMMs, fp64
CholeskyQR + the small SVD, the three quantised recombination GEMMs).  Default workload:
BASELINE configs[2] (c3: m = n = k = 8192, r = 512, p = 32, q = 2, polynomial spectrum,
int4 packed per-row sketch Y = A.Omega, int8 power / projection / recombination), the largest
configuration that fits one GPU; c1, c2, c4, c5 via --config.

`value`  = effective approx-GEMM TOPS = 2 m n k * steps * world / (max-over-ranks device
           time), inputs resident in HBM, each step replayed from one captured CUDA graph;
`e2e`    = the same metric through the drop-in public API `lramm(numpy A, numpy B, params)`,
           which calls the C-ABI host entry `lramm_host_lramm`: host->device copies of A, B
           (pinned), the pipeline, and the device->host copy of D every step.
N > 1 ranks run independent pairs (c1-c4: one per rank, or the 64 c4 pairs sharded), or the
row/column-sharded single pair (c5).
`--impl reference` times the unmodified reference (installed into oracle/_ref, its "python"
backend = OpenBLAS on all host cores, the faster of its two backends) on the same config:
one reference lramm() call per step, the integer recombination products timed on a row slice
of their left operand and scaled so a c3 step takes ~30 s
instead of ~430 s.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# The pipeline forks each product into two rsvd chains plus helper streams; with the default 8
# hardware work queues the streams of concurrent products alias onto the same queue and serialise
# (c4: 20.9 ms with 8 queues, 12.3 ms with 32).  Read at CUDA context creation.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

CONFIGS = {
    # BASELINE.json configs[1]
    "c2": dict(m=4096, k=4096, n=4096, rank=256, oversample=16, power_iters=1, bits=(8, 8, 8), tau=128.0,
               mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="row"),
    # BASELINE.json configs[3]: 64 independent 2048^3 pairs, r=128, p=10, q=0 (reference default),
    # int8 sketches with the reference's per-tensor quantiser; batch sharded across ranks
    "c4": dict(m=2048, k=2048, n=2048, rank=128, oversample=10, power_iters=0, bits=(8, 8, 8), tau=64.0,
               mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="tensor", pairs=64, streams=16),
    # BASELINE.json configs[0] (the reference's CPU-runnable case), for quick runs
    "c1": dict(m=1024, k=1024, n=1024, rank=64, oversample=10, power_iters=1, bits=(8, 8, 8), tau=32.0,
               mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="row"),
    # BASELINE.json configs[2]: polynomial spectrum, int4 per-row sketch Y = A.Omega, int8 elsewhere
    "c3": dict(m=8192, k=8192, n=8192, rank=512, oversample=32, power_iters=2, bits=(8, 8, 8), poly=1.5,
               mode="fast", sketch_bits=4, power_bits=8, proj_bits=8, granularity="row"),
    # BASELINE.json configs[4]: tall-skinny; at N > 1 A is row-sharded and B column-sharded
    # (paper_2405_16917_b200/sharded.py), at N = 1 the whole problem runs on one GPU
    "c5": dict(m=131072, k=8192, n=8192, rank=1024, oversample=32, power_iters=1, bits=(8, 8, 8), tau=256.0,
               mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="tensor", sharded=True),
}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spectrum_name(cfg):
    return f"poly:{cfg['poly']}" if "poly" in cfg else f"exp:{int(cfg['tau'])}"


def synth_pair(cfg, seed, device):
    """A = U diag(sigma) V^T, B likewise; Haar U, V (thin QR of seeded Gaussians, sign-fixed);
    sigma_i = exp(-i/tau) + 1e-4 or i^-alpha; stored fp32."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(0x1A3A * 1000 + seed)

    def haar(n, t):
        z = torch.randn(n, t, generator=g, device=device, dtype=torch.float64)
        q, r = torch.linalg.qr(z)
        return q * torch.sign(torch.diagonal(r))

    def mat(rows, cols):
        t = min(rows, cols)
        i = torch.arange(1, t + 1, device=device, dtype=torch.float64)
        sig = i ** (-cfg["poly"]) if "poly" in cfg else torch.exp(-i / cfg["tau"]) + 1e-4
        u = haar(rows, t)
        v = haar(cols, t)
        out = ((u * sig) @ v.T).to(torch.float32).contiguous()
        del u, v
        return out

    return mat(cfg["m"], cfg["k"]), mat(cfg["k"], cfg["n"])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def mark(self):
        return len(self.samples)

    def summary(self, start=0):
        rows = self.samples[start:] or self.samples
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        busy = [s for s in rows if s[0].replace(".", "").isdigit() and float(s[0]) > 600]
        rows = busy or rows
        sm = [float(s[0]) for s in rows if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in rows if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in rows for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "window": "nvidia-smi -lms 100 over the warm-up + timed graph replays (samples with SM clock > 600 MHz)"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------ roofline of the dominant kernel

def roofline_probe(L, ta, tb, params, reps=5, step=None):
    """Time the hot path's kernels live (torch profiler over one step), pick the dominant one and
    express it against its roofline."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    step = step or (lambda: L.lramm_device(ta, tb, params))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            step()
        torch.cuda.synchronize()
    per = {}
    launches = 0
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        name = ev.name
        if "Memcpy" in name or "Memset" in name or "memcpy" in name or "memset" in name:
            continue
        launches += 1
        d = per.setdefault(name, [0.0, 0])
        d[0] += ev.device_time
        d[1] += 1
    total = sum(v[0] for v in per.values())
    if not per:  # no CUPTI events (e.g. running under ncu, which owns the profiler)
        return "unavailable (profiler busy)", 0.0, 0, 0.0, 0, per
    top = max(per.items(), key=lambda kv: kv[1][0])
    return top[0], top[1][0] / top[1][1], top[1][1] // reps, total / reps, launches // reps, per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true", help="skip the report-only accuracy checks")
    ap.add_argument("--sharded", action="store_true",
                    help="run the row/column-sharded path (the default at N > 1 for a single pair) even at N = 1")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: one independent pair per rank (no collective) instead of the sharded pair")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)
    # N > 1: a single pair is row/column-sharded over the ranks (north_star (4)); the batched
    # config shards its pairs instead; --replicas runs one independent pair per rank
    if args.sharded or (world > 1 and cfg.get("pairs", 1) == 1 and not args.replicas):
        return run_sharded(args, cfg, world, rank, local)
    return run_ours(args, cfg, world, rank, local)


def effective_ops(cfg):
    return 2.0 * cfg["m"] * cfg["n"] * cfg["k"]


def pairs_per_rank(cfg, world):
    total = cfg.get("pairs", 1)
    if total == 1:
        return 1
    if total % world:
        raise SystemExit(f"{total} pairs do not shard evenly over {world} ranks")
    return total // world


def workload_config(cfg, args, world):
    total = cfg.get("pairs", 1)
    which = {"c1": "configs[0]", "c2": "configs[1]", "c3": "configs[2]", "c4": "configs[3]",
             "c5": "configs[4]"}[args.config]
    sharded = world > 1 and total == 1 and not getattr(args, "replicas", False)
    return {"workload": f"BASELINE {which}: {total} x {cfg['m']}x{cfg['k']}x{cfg['n']} fp32 {spectrum_name(cfg)} "
                        f"spectrum, r={cfg['rank']} p={cfg['oversample']} q={cfg['power_iters']}, "
                        f"int{cfg['sketch_bits']}/int{cfg['power_bits']}/int{cfg['proj_bits']} "
                        f"{cfg['granularity']}-scaled sketch/power/projection GEMMs, recombination bits {cfg['bits']}",
            "name": args.config, "m": cfg["m"], "k": cfg["k"], "n": cfg["n"], "rank": cfg["rank"],
            "oversample": cfg["oversample"], "power_iters": cfg["power_iters"], "bits": list(cfg["bits"]),
            "mode": cfg["mode"], "granularity": cfg["granularity"], "pairs_per_rank": pairs_per_rank(cfg, world),
            "streams": min(pairs_per_rank(cfg, world), int(os.environ.get("BENCH_STREAMS", cfg.get("streams", 1)))),
            "graphs": max(1, min(pairs_per_rank(cfg, world), int(os.environ.get("BENCH_GRAPHS", cfg.get("graphs", 1))))),
            "parallelism": (f"{world} ranks, A row-sharded / B column-sharded, NCCL Gram + int32 partial "
                            f"allreduces, E2 allgather" if sharded else
                            f"{world} ranks, independent pairs sharded across ranks (no collective)" if world > 1
                            else "single GPU"),
            "l2": f"inputs ({(cfg['m'] * cfg['k'] + cfg['k'] * cfg['n']) * 4 / 2**20:.0f} MiB fp32) exceed the "
                  f"126 MB L2; no explicit flush"}


E_SAMPLE_ROWS = 128  # rows of each recombination product's left operand timed through _kernels.imatmul


def import_reference():
    """The unmodified reference package from oracle/_ref with its "python" kernel backend
    (LRAMM_PURE_PYTHON=1: LAPACK / OpenBLAS on all host cores), the faster of its two backends
    (c2 22.6 s vs 64.7 s compiled)."""
    os.environ["LRAMM_PURE_PYTHON"] = "1"
    path = os.path.join(ROOT, "oracle", "_ref")
    if path not in sys.path:
        sys.path.insert(0, path)
    import lramm as ref  # noqa: E402

    return ref


def reference_step(ref, a, b, cfg, sample_rows=E_SAMPLE_ROWS):
    """One reference lramm() call on (a, b), statement by statement through the reference's own
    functions (pipeline.py:159-214): rsvd(A), rsvd(B) (rsvd.py:68-81, the oracle size cap raised
    at call time for w > 512), the scaling block, and the three QM products
    (quant.qgemm, quant.py:96-121) whose integer product _kernels.imatmul is row-separable: it is
    timed on the first `sample_rows` rows of the left operand and scaled to the full row count
    (SURVEY §8(d)); quantize, the overflow check and the dequantisation are timed in full.
    Returns (seconds, per-stage seconds, D): D from exact float64 products of the same integers
    (bit-identical to _kernels.imatmul while K cap^2 < 2^53; untimed)."""
    import lramm.matcore as rm
    from lramm import _kernels as rk
    from lramm import quant as rq
    import lramm.rsvd  # noqa: F401
    rr = sys.modules["lramm.rsvd"]  # the module: lramm re-exports the rsvd function under the same name
    from lramm.pipeline import _child_seeds

    r, q, p = cfg["rank"], cfg["power_iters"], cfg["oversample"]
    w = min(r + p, *a.shape, *b.shape)
    rm.ORACLE_MAX_MIN_DIM = max(512, w)  # harness override of the module constant (matcore.py:23)
    params = ref.LrammParams(rank=r, bits=tuple(cfg["bits"]), power_iters=q, oversample=p, seed=0)
    d1, d2, d3 = params.bits
    a = rm.as_matrix(a, "a")
    b = rm.as_matrix(b, "b")
    seed_a, seed_b = _child_seeds(params.seed)
    st = {}
    t0 = time.perf_counter()
    fa = rr.rsvd(a, rr.RsvdParams(params.rank, params.power_iters, params.oversample, seed_a))
    fb = rr.rsvd(b, rr.RsvdParams(params.rank, params.power_iters, params.oversample, seed_b))
    st["rsvd"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    u_scaled = np.ascontiguousarray(fa.u * fa.sigma)
    z_scaled = np.ascontiguousarray((fb.v * fb.sigma).T)
    vt = np.ascontiguousarray(fa.v.T)
    wq = fb.u
    st["scaling"] = time.perf_counter() - t0

    def qm(x, y, bits):
        t0 = time.perf_counter()
        qx, qy = rq.quantize(x, bits), rq.quantize(y, bits)
        rq._check_overflow(x.shape[1], bits, bits)
        t_full = time.perf_counter() - t0
        rows = min(sample_rows, x.shape[0])
        t0 = time.perf_counter()
        part = rk.imatmul(np.ascontiguousarray(qx.data[:rows]), qy.data)
        _ = part.astype(np.float64) / (qx.scale * qy.scale)
        t_rows = time.perf_counter() - t0
        exact = (qx.data.astype(np.float64) @ qy.data.astype(np.float64)) / (qx.scale * qy.scale)
        return exact, t_full + t_rows * x.shape[0] / rows

    e1, st["gemm1"] = qm(vt, wq, d1)
    e2, st["gemm2"] = qm(e1, z_scaled, d2)
    d, st["gemm3"] = qm(u_scaled, e2, d3)
    return sum(st.values()), st, d


def reference_sample_note(cfg, pairs=1):
    rows = min(E_SAMPLE_ROWS, cfg["m"])
    return (f"{pairs} x one reference lramm() call per step on the same inputs (backend python: LAPACK + OpenBLAS "
            f"on all host cores), statement by statement (pipeline.py:159-214); the integer products of gemm1/2/3 "
            f"timed on the first {min(E_SAMPLE_ROWS, cfg['rank'])} / {min(E_SAMPLE_ROWS, cfg['rank'])} / {rows} "
            f"rows of their left operand and scaled to the full row count (row-separable, SURVEY §8(d)); "
            f"oracle SVD cap raised to the sketch width (SURVEY K5)")


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return 0
    try:
        ref = import_reference()
    except Exception as exc:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": f"reference not importable: {exc}"}))
        return 0
    import torch

    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    a, b = synth_pair(cfg, 0, dev)  # input synthesis only (the reference itself runs on the host)
    a, b = a.cpu().numpy(), b.cpu().numpy()
    pairs = cfg.get("pairs", 1)
    steps = max(1, min(args.steps, 2))
    times, stages = [], None
    for _ in range(steps):
        t, stages, _d = reference_step(ref, a, b, cfg)
        times.append(t * pairs)  # c4: the 64 pairs are identical in cost (one timed, scaled)
    t = float(np.mean(times))
    value = effective_ops(cfg) * pairs / t / 1e12
    cores = os.cpu_count()
    line = {"metric": "effective approx-GEMM TOPS (2mnk/time)", "value": value, "unit": "TOPS", "n_gpus": args.gpus,
            "steps": steps, "warmup": 0, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64 (fp32 inputs upcast), int64 QM products", "data": "synthetic",
            "impl": "reference", "config": workload_config(cfg, args, 1),
            "stages_s": stages,
            "cpu_baseline": {"value": value, "unit": "TOPS", "cores": cores, "kind": "reference",
                             "sample": reference_sample_note(cfg, pairs) + f"; {steps} step(s), no warm-up"},
            "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args, cfg, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    import paper_2405_16917_b200 as L

    P = pairs_per_rank(cfg, world)
    S = min(P, int(os.environ.get("BENCH_STREAMS", cfg.get("streams", 1))))
    pairs = [synth_pair(cfg, rank * P + j, dev) for j in range(P)]
    a, b = pairs[0]
    params = L.LrammParams(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"],
                           oversample=cfg["oversample"], seed=rank, mode=cfg["mode"], sketch_bits=cfg["sketch_bits"],
                           power_bits=cfg["power_bits"], proj_bits=cfg["proj_bits"], granularity=cfg["granularity"],
                           out_dtype=np.float32)
    outs = [torch.empty((cfg["m"], cfg["n"]), dtype=torch.float32, device=dev) for _ in range(P)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(S)]

    def issue_all():
        """All pairs of this rank: pair j on stream j % S (each stream has its own workspace)."""
        cur = torch.cuda.current_stream(dev)
        evs = []
        for st_ in streams:
            st_.wait_stream(cur)
        for j, (aj, bj) in enumerate(pairs):
            with torch.cuda.stream(streams[j % S]):
                _o, status_j, _t = L.lramm_device(aj, bj, params, out=outs[j])
        for st_ in streams:
            cur.wait_stream(st_)
        return status_j

    clocks = ClockSampler(local).__enter__()
    time.sleep(0.5)  # nvidia-smi start-up
    # warm-up (also sets kernel attributes and allocates per-stream workspaces before capture)
    for _ in range(max(1, args.warmup)):
        status = issue_all()
    torch.cuda.synchronize()
    st = int(status.item())
    if st:
        raise RuntimeError(f"lramm status {st}")
    # capture one step (all pairs of this rank) into a CUDA graph -- or, for the batched config, into
    # BENCH_GRAPHS graphs (pairs split evenly) replayed side by side on their own launch streams
    G = max(1, min(P, int(os.environ.get("BENCH_GRAPHS", cfg.get("graphs", 1)))))
    groups = [list(range(g, P, G)) for g in range(G)]

    def issue_group(g):
        cur = torch.cuda.current_stream(dev)
        mine = streams[g::G] if S >= G else [streams[g % S]]
        for st_ in mine:
            st_.wait_stream(cur)
        for i, j in enumerate(groups[g]):
            with torch.cuda.stream(mine[i % len(mine)]):
                L.lramm_device(pairs[j][0], pairs[j][1], params, out=outs[j])
        for st_ in mine:
            cur.wait_stream(st_)

    caps = [torch.cuda.Stream(device=dev) for _ in range(G)]
    graphs = [torch.cuda.CUDAGraph() for _ in range(G)]
    for g in range(G):
        caps[g].wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(caps[g]):
            if G == 1:
                issue_all()
            else:
                issue_group(g)
            torch.cuda.synchronize()
            with torch.cuda.graph(graphs[g], stream=caps[g]):
                if G == 1:
                    issue_all()
                else:
                    issue_group(g)
    torch.cuda.synchronize()

    class _Replay:
        def replay(self):
            if G == 1:
                graphs[0].replay()
                return
            cur = torch.cuda.current_stream(dev)
            for g in range(G):
                caps[g].wait_stream(cur)
                with torch.cuda.stream(caps[g]):
                    graphs[g].replay()
            for g in range(G):
                cur.wait_stream(caps[g])

    graph = _Replay()
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk_mark = clocks.mark()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # keep the GPU busy with more replays (untimed) so the sampler sees the loaded clocks
    t_end = time.time() + 1.0
    while time.time() < t_end:
        graph.replay()
        torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    clock_summary = clocks.summary(clk_mark)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    ms_per_step = ms / args.steps
    value = effective_ops(cfg) * P * world / (ms_per_step * 1e-3) / 1e12

    # ---- e2e through the drop-in public API (host buffers, C-ABI host entry point)
    host_pairs = []
    for aj, bj in pairs:
        ha = torch.empty(aj.shape, dtype=torch.float32, pin_memory=True)
        hb = torch.empty(bj.shape, dtype=torch.float32, pin_memory=True)
        ha.copy_(aj.cpu())
        hb.copy_(bj.cpu())
        host_pairs.append((ha.numpy(), hb.numpy()))
    p64 = L.LrammParams(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"],
                        oversample=cfg["oversample"], seed=rank, mode=cfg["mode"], sketch_bits=cfg["sketch_bits"],
                        power_bits=cfg["power_bits"], proj_bits=cfg["proj_bits"], granularity=cfg["granularity"])
    # P > 1 (batched pairs): the pairs are issued from a pool of host threads, each call on its own
    # leased C-ABI context and streams (the reference's sweeps use a thread pool the same way,
    # cli.py:415-419); per-thread pinned D buffers
    # P == 1: INFLIGHT calls are kept in flight from as many host threads, so call i+1's upload and
    # call i-1's download overlap call i's factorisation (PCIe is full duplex and each call leases its
    # own context); every call still moves its own A, B up and its own D down inside the timed region.
    # The latency of one isolated call is reported next to the throughput.
    inflight = max(1, int(os.environ.get("BENCH_E2E_INFLIGHT", 3)))
    workers = min(P, 8) if P > 1 else inflight
    tls = threading.local()

    def host_call(pair):
        if not hasattr(tls, "out"):
            tls.out = torch.empty((cfg["m"], cfg["n"]), dtype=torch.float64, pin_memory=True).numpy()
        torch.cuda.set_device(local)
        return L.lramm(pair[0], pair[1], p64, out=tls.out)

    from concurrent.futures import ThreadPoolExecutor

    pool = ThreadPoolExecutor(max_workers=workers)
    calls = host_pairs if P > 1 else host_pairs * (inflight * int(os.environ.get("BENCH_E2E_ROUNDS", 6)))
    for _ in range(max(1, min(args.warmup, 2))):
        list(pool.map(host_call, (host_pairs * workers)[:workers]))
    e2e_steps = max(1, min(args.steps, 5 if P == 1 else 1))
    lat_s = None
    if P == 1:  # one isolated call at a time
        host_call(host_pairs[0])  # this thread's pinned D buffer
        t0 = time.perf_counter()
        for _ in range(3):
            host_call(host_pairs[0])
        lat_s = (time.perf_counter() - t0) / 3
        e2e_steps = 1
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        list(pool.map(host_call, calls))
    e2e_s = (time.perf_counter() - t0) / e2e_steps / (len(calls) // P)
    pool.shutdown()
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    wa = min(cfg["rank"] + cfg["oversample"], cfg["k"])
    # A and B cross PCIe every step; Omega is generated on the device from the seed (lramm_omega)
    h2d = P * 4 * (cfg["m"] * cfg["k"] + cfg["k"] * cfg["n"])
    d2h = P * 8 * cfg["m"] * cfg["n"]
    e2e = {"value": effective_ops(cfg) * P * world / e2e_s / 1e12, "unit": "TOPS", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
           "path": "lramm(numpy) -> lramm_host_lramm (C ABI), pinned A/B/D, fp64 D like the reference; "
                   "Omega from the device generator (cached per seed)"
                   + (f"; pairs issued from {workers} host threads" if P > 1 else
                      f"; {len(calls)} calls, {inflight} in flight from {inflight} host threads (throughput); "
                      "single_call_ms = one isolated call")}
    if lat_s is not None:
        e2e["single_call_ms"] = lat_s * 1e3
        e2e["single_call_value"] = effective_ops(cfg) * world / lat_s / 1e12
        e2e["calls_in_flight"] = inflight

    # ---- dominant kernel + launches (live, torch profiler over device-resident steps)
    top_name, top_us, top_per_step, step_us, launches, per = roofline_probe(L, a, b, params)
    launches *= P  # per step = all pairs of this rank
    peaks = measured_peaks()
    peaks["live"] = measure_peaks(dev)
    roof = dominant_roofline(top_name, top_us, cfg, peaks)
    roof["kernel"] = top_name
    roof["us_per_launch"] = top_us
    roof["launches_per_step"] = top_per_step
    roof["share_of_step"] = top_us * top_per_step / step_us if step_us else None
    stages = stage_rooflines(per, 5, cfg, peaks) if per else None

    def _short(nm):
        return nm.replace("lramm::(anonymous namespace)::", "").replace("void ", "").split("(")[0]

    top_kernels = [{"kernel": _short(nm), "us_per_step": v[0] / 5, "launches_per_step": v[1] // 5}
                   for nm, v in sorted(per.items(), key=lambda kv: -kv[1][0])[:14]] if per else None

    line = {"metric": "effective approx-GEMM TOPS (2mnk/time)", "value": value, "unit": "TOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "int8 x int8 -> int32 (tcgen05) sketch/QM GEMMs; fp64 factorisation; fp32 D",
            "data": "synthetic (SURVEY §8(d) spectrum, Haar factors from seeded torch QR)",
            "config": workload_config(cfg, args, world), "clocks": clock_summary, "e2e": e2e,
            "gpu_launches": launches * args.steps, "gpu_launches_per_step": launches, "roofline": roof,
            "stages": stages, "top_kernels": top_kernels, "peaks": peaks.get("live")}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], d_ref = cpu_baseline(cfg, a, b)
    else:
        d_ref = None
    if rank == 0 and not args.no_accuracy:
        line["accuracy"] = accuracy(L, cfg, a, b, outs[0], params, d_ref)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_sharded(args, cfg, world, rank, local):
    """One approximate GEMM per step with A row-sharded and B column-sharded over the ranks
     through the C-ABI entry lramm_lramm_sharded: NCCL allreduces of the Gram
    matrices, the int32 partial accumulators and the quantiser maxima, one int8 allgather; the
    whole step captured in a CUDA graph.  value = 2mnk / (max-over-ranks device time), strong
    scaling.  At N = 1 (--sharded) the collectives still go through NCCL (single-rank
    communicators) so the line measures the same code path."""
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    import paper_2405_16917_b200 as L
    from paper_2405_16917_b200.sharded import NcclComm, lramm_sharded_native, shard_bounds

    m, k, n = cfg["m"], cfg["k"], cfg["n"]
    a, b = synth_pair(cfg, 0, dev)  # same seed on every rank: each keeps its own slice
    (ma, mb), (na, nb) = shard_bounds(m, n, world, rank)
    a_i, b_j = a[ma:mb].contiguous(), b[:, na:nb].contiguous()
    del a, b
    torch.cuda.empty_cache()
    kw = dict(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"], oversample=cfg["oversample"],
              seed=0, mode=cfg["mode"], sketch_bits=cfg["sketch_bits"], power_bits=cfg["power_bits"],
              proj_bits=cfg["proj_bits"], granularity=cfg["granularity"])
    params = L.LrammParams(out_dtype=np.float32, **kw)
    # two communicators let the A and B chains run concurrently; across ranks that is only safe when
    # NCCL's kernels and ours can always be co-resident, so the default at N > 1 is one communicator
    # (chains one after the other); SHARDED_TWO_COMMS=1 opts in
    two = world == 1 or os.environ.get("SHARDED_TWO_COMMS", "0") == "1"
    # NCCL prints its version banner on stdout at communicator creation: keep stdout for the JSON line
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        comm = NcclComm(force=(world == 1), two_comms=two)
        torch.cuda.synchronize()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    out = torch.empty((mb - ma, n), dtype=torch.float32, device=dev)

    def step():
        return lramm_sharded_native(a_i, b_j, (m, k, n), params, comm, out=out)

    clocks = ClockSampler(local).__enter__()
    time.sleep(0.5)
    for _ in range(max(1, args.warmup)):
        _d, status = step()
    torch.cuda.synchronize()
    st = int(status.item())
    if st:
        raise RuntimeError(f"lramm_sharded status {st}")
    # capture one step (kernels + NCCL collectives) into a CUDA graph
    cap = torch.cuda.Stream(device=dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap):
        step()  # sizes this stream's workspace
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=cap):
            step()
    torch.cuda.synchronize()
    for _ in range(max(3, args.warmup)):
        graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk_mark = clocks.mark()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    # keep the GPU loaded for the clock sampler (untimed): the SAME number of replays on every rank
    # (each replay contains collectives), derived from the all-reduced step time
    for _ in range(int(min(500, max(1, 1000.0 / max(ms_per_step, 1e-3))))):
        graph.replay()
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    clock_summary = clocks.summary(clk_mark)
    if world > 1:
        torch.distributed.barrier()
    value = effective_ops(cfg) / (ms_per_step * 1e-3) / 1e12

    # e2e: this rank's shards from pinned host memory, its fp64 D rows back to the host, every step
    p64 = L.LrammParams(**kw)
    ha = torch.empty(a_i.shape, dtype=torch.float32, pin_memory=True)
    hb = torch.empty(b_j.shape, dtype=torch.float32, pin_memory=True)
    ha.copy_(a_i)
    hb.copy_(b_j)
    hd = torch.empty((mb - ma, n), dtype=torch.float64, pin_memory=True)
    d64 = torch.empty((mb - ma, n), dtype=torch.float64, device=dev)
    e2e_steps = max(1, min(args.steps, 3))

    def e2e_step():
        da, db = ha.to(dev, non_blocking=True), hb.to(dev, non_blocking=True)
        lramm_sharded_native(da, db, (m, k, n), p64, comm, out=d64)
        hd.copy_(d64)

    e2e_step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": effective_ops(cfg) / e2e_s / 1e12, "unit": "TOPS",
           "h2d_bytes_per_step": 4 * (a_i.numel() + b_j.numel()), "d2h_bytes_per_step": 8 * hd.numel(),
           "ms_per_step": e2e_s * 1e3,
           "path": "lramm_sharded_native (C ABI lramm_lramm_sharded) on this rank's pinned host shards, fp64 D rows"}
    top_name, top_us, top_per_step, step_us, launches, per = roofline_probe(L, None, None, None, reps=2, step=step)
    peaks = measured_peaks()
    if rank == 0:
        peaks["live"] = measure_peaks(dev)
    roof = dominant_roofline(top_name, top_us, cfg, peaks)
    roof.update(kernel=top_name, us_per_launch=top_us, launches_per_step=top_per_step,
                share_of_step=top_us * top_per_step / step_us if step_us else None)
    nccl = [(us, c) for name, (us, c) in per.items() if "nccl" in name.lower()] if per else []
    nccl_us = sum(us for us, _c in nccl) / 2 if per else None
    launches -= sum(c for _us, c in nccl) // 2  # gpu_launches counts this library's kernels only
    line = {"metric": "effective approx-GEMM TOPS (2mnk/time)", "value": value, "unit": "TOPS", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "int8 x int8 -> int32 (tcgen05) sketch/QM GEMMs; fp64 factorisation; fp32 D",
            "data": "synthetic (SURVEY §8(d) spectrum, Haar factors from seeded torch QR)",
            "config": dict(workload_config(cfg, args, world), parallelism=(
                f"{world} ranks, A row-sharded / B column-sharded (lramm_lramm_sharded): NCCL allreduce of Gram "
                f"matrices, int32 partial accumulators and quantiser maxima, int8 E2 allgather; "
                f"{'two communicators, concurrent A/B chains' if two else 'one communicator, A then B chain'}; "
                f"one CUDA graph per step" + ("" if world > 1 else "; single-rank NCCL communicators"))),
            "clocks": clock_summary, "e2e": e2e, "gpu_launches": launches * args.steps,
            "gpu_launches_per_step": launches, "roofline": roof, "nccl_us_per_step": nccl_us,
            "peaks": peaks.get("live")}
    if rank == 0:
        print(json.dumps(line))
    comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


# dram__bytes_read.sum + dram__bytes_write.sum per launch from `ncu --set full` captures
# (profiles/r01_ncu_jacobi_c2.txt)
NCU_DRAM_BYTES = {  # dram__bytes_read.sum + dram__bytes_write.sum of one launch, ncu --set full
    "jacobi_cluster_kernel<9, false>": 639488,  # profiles/r01_ncu_jacobi_c2.txt
    "sytrd_push_kernel<17, 0>": 2426624,        # profiles/r02_ncu_sytrd_c3.txt (the one load of the Gram matrix)
}


FP64_PEAK_SOURCE = "fp64 DGEMM 8192^3 measured live in this run (peaks.live.fp64_tflops)"


def fp64_peak_tflops(peaks):
    """fp64 tensor peak: measured live (cuBLAS DGEMM) in this run, else the DMMA microbenchmark
    of profiles/r01_fp64_peak.txt (36.7)."""
    v = (peaks.get("live") or {}).get("fp64_tflops")
    return float(v) if v else 36.7


def int8_peak_tops(peaks):
    """int8 tensor peak: measured live (torch._int_mm 8192^3) in this run, else nominal 4500."""
    v = (peaks.get("live") or {}).get("int8_tops")
    return float(v) if v else 4500.0


def dominant_roofline(name, us, cfg, peaks):
    """Algorithmic work of the dominant kernel per launch over its measured time."""
    if not us:
        return {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None}
    m, k, n, r = cfg["m"], cfg["k"], cfg["n"], cfg["rank"]
    w = r + cfg["oversample"]
    fp64_peak = fp64_peak_tflops(peaks)
    if "jacobi" in name:
        # one-sided Jacobi on the w x w R^T: sweeps x w(w-1)/2 pairs x 8w flops (dot product 2w +
        # rotation 6w); sweeps measured by scripts/sweeps_probe.py: 9 (c1-c3), 10 (c5)
        sweeps = 10 if w > 1000 else 9
        flops = sweeps * (w * (w - 1) / 2) * 8 * w
        achieved = flops / (us * 1e-6) / 1e12
        traffic = next((v for k, v in NCU_DRAM_BYTES.items() if k in name), None)
        return {"bound": "tensor", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": traffic, "algorithmic_flops": flops,
                "peak_source": FP64_PEAK_SOURCE,
                "note": "latency-bound sequential rotation chain (w steps per sweep); traffic: columns stay in "
                        "shared memory, DRAM bytes are the one-time load of R^T"}
    if "sytrd" in name:
        # Householder tridiagonalisation of the w x w Gram R R^T (the eigenvector preconditioner of the
        # small SVD): 4/3 w^3 flops in w - 2 dependent steps
        flops = 4.0 / 3.0 * w ** 3
        achieved = flops / (us * 1e-6) / 1e12
        traffic = next((v for k, v in NCU_DRAM_BYTES.items() if k in name), None)
        return {"bound": "tensor", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": traffic, "algorithmic_flops": flops,
                "peak_source": FP64_PEAK_SOURCE, "class": "latency-bound (CUDA-core fp64, not a throughput kernel)",
                "note": "latency-bound: w - 2 dependent reflector steps, each one DSMEM exchange (st.async + "
                        "mbarrier) across the cluster; the matrix stays in registers / shared memory (no DRAM "
                        "traffic beyond the one load of the Gram matrix)"}
    if "chol" in name or "trinv" in name:
        flops = w ** 3 / 3.0
        achieved = flops / (us * 1e-6) / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": None,
                "peak_source": FP64_PEAK_SOURCE + "; kernel is latency-bound"}
    if "dgemm" in name:
        flops = 2.0 * m * w * w
        achieved = flops / (us * 1e-6) / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": None, "peak_source": FP64_PEAK_SOURCE}
    # int8 tcgen05 GEMM / quantiser: HBM-bound at these shapes
    hbm = peaks.get("hbm_gbs", 6538.0)
    byts = m * k * 1 + w * k * 1 + m * w * 8
    achieved = byts / (us * 1e-6) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}


STAGES = (  # kernel-name fragments -> stage of the hot path
    ("omega", ("omega",)),
    ("quantize", ("absmax", "quantize", "scales_from", "split_limbs")),
    ("int8_gemm", ("igemm", "epilogue")),
    ("small_svd", ("jacobi", "col_norms", "rank_kernel", "finalize_write", "complete_kernel", "scale_cols", "sytrd",
                   "bisect", "twisted", "reflector_t", "backtransform", "eig_defect", "refine_", "offrel",
                   "copy_if_converged")),
    ("fp64_qr", ("dgemm", "chol", "trsm", "cf_prep", "splitk", "transpose", "householder", "diag_inv",
                 "set_identity", "any_nonzero")),
)


def stage_rooflines(per, reps, cfg, peaks, sweeps=10):
    """Per-stage device time (kernel time summed over both operand chains, per step) against the
    stage's roofline time max(ops / peak, bytes / HBM) from its algorithmic work."""
    m, k, n, r, q = cfg["m"], cfg["k"], cfg["n"], cfg["rank"], cfg["power_iters"]
    w = min(r + cfg["oversample"], m, k, n)
    hbm = peaks.get("hbm_gbs", 6538.0) * 1e9
    fp64 = fp64_peak_tflops(peaks) * 1e12
    int8 = int8_peak_tops(peaks) * 1e12
    # quantiser: fp32 operands read once, two int8 copies written; fp64 sketch/recombination operands 8 B + 1 B
    q_bytes = 6 * (m * k + k * n) + 9 * ((k * w + q * (m * w + k * w) + m * w) + (n * w + q * (k * w + n * w) + k * w)
                                         + (r * k + k * r) + (r * r + r * n) + (m * r + r * n))
    prods = [(m, w, k, 8)] * (1 + q) + [(k, w, m, 8)] * (q + 1) + [(k, w, n, 8)] * (1 + q) + [(n, w, k, 8)] * (q + 1)
    prods += [(r, r, k, 8), (r, n, r, 8), (m, n, r, 4)]
    g_ops = sum(2.0 * M * N * K for M, N, K, _ in prods)
    g_bytes = sum(M * K + N * K + M * N * ob for M, N, K, ob in prods)
    # one CholeskyQR pass = Gram (2 rows w^2, full) + TRSM (rows w^2); parity mode and the SVD's
    # projection always run the second pass, fast-mode sketches only when kappa(Y) > ~95:
    # the minimum (one pass for fast-mode sketches) is the algorithmic work counted here
    sk_rows = [m] * (1 + q) + [k] * q + [k] * (1 + q) + [n] * q
    pj_rows = [k, n]
    passes = 1 if cfg.get("mode") == "fast" else 2
    qr_flops = (sum(3.0 * passes * rr * w * w for rr in sk_rows) + sum(6.0 * rr * w * w for rr in pj_rows)
                + 2.0 * (m + k) * w * w + 2.0 * (k + n) * w * w)
    # small SVD (per operand): tridiagonalisation 4/3 w^3, back-transform 2 w^3, the Gram / Lowdin /
    # rotation / check GEMMs 5 x 2 w^3 (the refinement GEMMs only run when the check fails)
    svd_flops = 2 * (4.0 / 3.0 + 2.0 + 10.0) * w ** 3
    work = {
        "omega": (0.0, 8.0 * (k + n) * w, "bytes: Omega_A, Omega_B written (fp64)"),
        "quantize": (0.0, float(q_bytes), "bytes: fp32 operands read once + 2 int8 copies; fp64 sketch and "
                                         "recombination operands read + int8 written"),
        "int8_gemm": (g_ops / int8, float(g_bytes), "2MNK over the sketch/projection/recombination products; "
                                                   "int8 operands read + outputs written"),
        "fp64_qr": (qr_flops / fp64, 0.0, "3 rows w^2 per CholeskyQR pass (one pass for fast-mode sketches, two "
                                          "for the projections) + the two lifts (fp64 tensor peak)"),
        "small_svd": (svd_flops / fp64, 0.0, "eigenvector-preconditioned SVD of the w x w R^T, two operands: "
                                            "tridiagonalisation 4/3 w^3 + back-transform 2 w^3 + 5 GEMMs 2 w^3"),
    }
    out = {}
    for stage, frags in STAGES:
        us = sum(v[0] for name, v in per.items() if any(f in name for f in frags)) / reps
        t_ops, byts, what = work[stage]
        roof_us = max(t_ops, byts / hbm) * 1e6
        out[stage] = {"us_per_step": us, "roofline_us": roof_us, "frac": (roof_us / us) if us else None,
                      "bound": "hbm" if byts / hbm >= t_ops else ("int8 tensor" if stage == "int8_gemm" else "fp64"),
                      "work": what}
    known = sum(v["us_per_step"] for v in out.values())
    out["other"] = {"us_per_step": sum(v[0] for v in per.values()) / reps - known}
    out["note"] = ("kernel time summed over the concurrent A/B chains (torch profiler over device-resident steps, "
                   "outside the timed region); frac = roofline time / measured time")
    return out


def cpu_baseline(cfg, a, b):
    """The unmodified reference (oracle/_ref) timed on this host: one sampled reference step on
    the same inputs (reference_step)."""
    try:
        ref = import_reference()
    except Exception as exc:
        return {"value": None, "unit": "TOPS", "cores": os.cpu_count(), "kind": "reference",
                "sample": f"unavailable: {exc}"}, None
    ha, hb = a.cpu().numpy(), b.cpu().numpy()
    t, stages, d_ref = reference_step(ref, ha, hb, cfg)
    pairs = cfg.get("pairs", 1)
    return {"value": effective_ops(cfg) * pairs / (t * pairs) / 1e12, "unit": "TOPS", "cores": os.cpu_count(),
            "kind": "reference", "seconds_per_call": t, "stages_s": stages,
            "sample": reference_sample_note(cfg, 1) + (f"; one of the {pairs} pairs (identical cost)" if pairs > 1 else "")
            }, d_ref


def measure_peaks(dev):
    """Live tensor-pipe peaks on this box (cuBLAS, 8192^3, best of 10, CUDA events): int8 x int8 ->
    int32 (torch._int_mm) and fp64 DGEMM, the roofline denominators MEASURED_PEAKS.json lacks."""
    import torch

    out = {}
    n = 8192
    for name, mk, flops in (("int8_tops", lambda: torch._int_mm, 2.0 * n ** 3),
                            ("fp64_tflops", lambda: torch.matmul, 2.0 * n ** 3)):
        try:
            if name == "int8_tops":
                x = torch.randint(-127, 128, (n, n), dtype=torch.int8, device=dev)
                y = torch.randint(-127, 128, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
            else:
                x = torch.randn(n, n, dtype=torch.float64, device=dev)
                y = torch.randn(n, n, dtype=torch.float64, device=dev)
            fn = mk()
            for _ in range(3):
                fn(x, y)
            best = 1e30
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn(x, y)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            out[name] = flops / (best * 1e-3) / 1e12
            del x, y
        except Exception as exc:  # pragma: no cover
            out[name] = None
            out[name + "_error"] = str(exc)[:200]
    out["how"] = "cuBLAS 8192^3 (torch._int_mm int8->int32; torch.matmul fp64), best of 10, CUDA events, in this run"
    return out


def accuracy(L, cfg, a, b, d_ours, params, d_ref=None):
    """Report only, after the timed region: the benchmarked (fast-mode) product against
    (1) the CPU restatement of the same fast-mode algorithm (the L5 parity gate, <= 1e-3),
    (2) the exact fp64 product, next to the reference's own error on the same inputs, and
    (3) the reference's output (where the reference step ran): this package's parity-mode
    product (the reference's algorithm: fp64 sketches, per-tensor QM) against it (<= 1e-9 gate)."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lramm_oracle as O  # the checker (test infrastructure), never the thing measured

    exact = a.double() @ b.double()
    nrm = torch.linalg.norm(exact)
    out = {"rel_err_vs_exact": float(torch.linalg.norm(d_ours.double() - exact) / nrm),
           "exact": "fp64 product of the same fp32 inputs (cuBLAS DGEMM, report only)"}
    ha, hb = a.cpu().numpy(), b.cpu().numpy()
    kw = dict(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"],
              oversample=cfg["oversample"], seed=int(params.seed))
    spec = O.SketchSpec(cfg["sketch_bits"], cfg["power_bits"], cfg["proj_bits"], cfg["granularity"])
    t0 = time.perf_counter()
    d_rest = torch.from_numpy(O.lramm(ha, hb, O.OracleParams(**kw, spec=spec))).to(exact.device)
    out["fast_mode_rel_diff_vs_restatement"] = float(torch.linalg.norm(d_ours.double() - d_rest) /
                                                     torch.linalg.norm(d_rest))
    if d_ours.dtype == torch.float32:  # the floor: D itself rounded to fp32
        out["fp32_rounding_of_restatement"] = float(torch.linalg.norm(d_rest.float().double() - d_rest) /
                                                    torch.linalg.norm(d_rest))
    out["restatement_s"] = time.perf_counter() - t0
    if d_ref is not None:
        dr = torch.from_numpy(np.ascontiguousarray(d_ref)).to(exact.device)
        e_ref = float(torch.linalg.norm(dr - exact) / nrm)
        out["reference_rel_err_vs_exact"] = e_ref
        out["fast_mode_error_within_2pct_of_reference"] = abs(out["rel_err_vs_exact"] - e_ref) <= 0.02 * e_ref
        p = L.LrammParams(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"],
                          oversample=cfg["oversample"], seed=int(params.seed))  # parity mode
        d_par, _, _ = L.lramm_device(a, b, p)
        out["parity_mode_rel_diff_vs_reference"] = float(torch.linalg.norm(d_par.double() - dr) / torch.linalg.norm(dr))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            L.lramm_device(a, b, p)
        e1.record()
        torch.cuda.synchronize()
        out["parity_mode_ms_per_step"] = e0.elapsed_time(e1) / 3
    out["note"] = ("fast mode (quantised sketches, the benchmarked path) is gated against its CPU restatement "
                   "(<= 1e-3) and on accuracy parity with the reference; the parity mode (the reference's "
                   "algorithm) is gated at <= 1e-9 against the reference's output")
    return out


if __name__ == "__main__":
    sys.exit(main())
