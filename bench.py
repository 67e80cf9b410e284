"""Benchmark of the TensorCommitments prover hot path on B200.

Default workload = BASELINE.json config 3 (the one the "prover overhead % vs 7B-shape
forward" metric is quoted on): 32 layers of LLaMA-2-7B-shaped hidden states
[1, 512, 4096] fp16 are quantised, committed (m = 4 grid (32,32,32,64)) and organised into
a 32-leaf Terkle tree (node shape (2,2,2)).  One step = one forward's prover work.  With
--gpus N (torchrun) the layers are partitioned over the ranks (strong scaling) and the
43-byte commitments all-gathered once.  `--config 5` runs the LLaMA-2-13B-shaped config
(40 layers [4,2048,5120], grid (64,128,64,80)); `--config 4` times batched openings.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3|4|5]

Prints ONE JSON line (rank 0).  `value` = field elements committed per second with the
activations resident in HBM; `e2e` = the same through the public API with the inputs
copied from pinned host memory and the commitments / root read back every step.
`--impl reference` times the CPU reference path (the oracle's CPython restatement of the
reference's arithmetic) on this host's cores over a bounded sample.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "field elems committed/sec; prover overhead % vs 7B-shape forward"
WORD_MULS_PER_ADD = 11 * 78   # 11 F_q mulmods per EC add, 78 word multiplies each
NODE_SHAPE = (2, 2, 2)
CONFIGS = {
    3: dict(layers=32, act=(1, 512, 4096), shape=(32, 32, 32, 64),
            name="config3: 32 layers x [1,512,4096] fp16 Student-t(3) x U(0.5,4) per layer, m=4 grid "
                 "(32,32,32,64), 32-leaf Terkle tree node shape (2,2,2)"),
    5: dict(layers=40, act=(4, 2048, 5120), shape=(64, 128, 64, 80),
            name="config5: 40 layers x [4,2048,5120] fp16 Student-t(3) x U(0.5,4) per layer, m=4 grid "
                 "(64,128,64,80), 40-leaf Terkle tree node shape (2,2,2)"),
}


def layer_scales(n_layers):
    import numpy as np
    return np.random.default_rng(12345).uniform(0.5, 4.0, n_layers)


def make_layers_host(cfg, layer_ids):
    """Seeded activations (host fp16): layer l = default_rng(l) standard_t(3) * scale_l."""
    import numpy as np
    scales = layer_scales(cfg["layers"])
    n = int(np.prod(cfg["act"]))
    out = []
    for l in layer_ids:
        x = np.random.default_rng(l).standard_t(3, size=n) * scales[l]
        out.append(x.astype(np.float16).reshape(cfg["act"]))
    return out


def make_layers_device(cfg, layer_ids, dev):
    """Config 5 is 1.7e9 values: generated on the GPU (torch Philox, seeded per layer)."""
    import torch
    scales = layer_scales(cfg["layers"])
    out = []
    for l in layer_ids:
        g = torch.Generator(device=dev).manual_seed(1000 + l)
        z = torch.randn(cfg["act"], generator=g, device=dev, dtype=torch.float32)
        # Student-t(3) = Z / sqrt(chi2_3 / 3), chi2_3 = sum of 3 squared normals
        c = sum(torch.randn(cfg["act"], generator=g, device=dev, dtype=torch.float32) ** 2 for _ in range(3))
        out.append((z / torch.sqrt(c / 3.0) * float(scales[l])).to(torch.float16))
    return out


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self, device=0):
        self.samples, self.proc, self.device = [], None, device

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)   # first sample lands before the timed region
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        num = lambda s: s.replace(".", "").isdigit()
        sm = [float(s[0]) for s in self.samples if num(s[0])]
        mx = [float(s[1]) for s in self.samples if num(s[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ 7B-shape forward
def forward_ms(device):
    """LLaMA-2-7B-shaped forward [1,512] with random fp16 weights (32 layers, hidden 4096,
    FFN 11008, vocab 32000, SDPA causal attention; RoPE omitted), CUDA-event timed."""
    import torch
    import torch.nn.functional as F
    torch.manual_seed(0)
    H, FF, V, L, S, NH = 4096, 11008, 32000, 32, 512, 32
    mk = lambda *s: (torch.randn(*s, device=device, dtype=torch.float16) * 0.02)
    emb = mk(V, H)
    layers = [(mk(3 * H, H), mk(H, H), mk(2 * FF, H), mk(H, FF)) for _ in range(L)]
    head = mk(V, H)
    ids = torch.randint(0, V, (1, S), device=device)

    def rms(x):
        return x * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-6).to(x.dtype)

    @torch.no_grad()
    def fwd():
        x = emb[ids]
        for wqkv, wo, wgu, wd in layers:
            h = rms(x)
            q, k, v = F.linear(h, wqkv).view(1, S, 3, NH, H // NH).permute(2, 0, 3, 1, 4)
            a = F.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(1, S, H)
            x = x + F.linear(a, wo)
            g, u = F.linear(rms(x), wgu).chunk(2, dim=-1)
            x = x + F.linear(F.silu(g) * u, wd)
        return F.linear(rms(x), head)

    for _ in range(3):
        fwd()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fwd()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    del layers, emb, head
    torch.cuda.empty_cache()
    return statistics.median(ts)


# ------------------------------------------------------------------ CPU reference leg
def _ref_modules():
    """(backend, field, mvpoly, kind): the unmodified reference copied into oracle/_ref by
    oracle/make_ref.py ("reference"), else the oracle's restatement ("port")."""
    from oracle import make_ref
    mods = make_ref.load()
    if mods is not None:
        return mods + ("reference",)
    return None, None, None, "port"


_TASK = None   # per-process sample (fork-inherited)


def _cpu_task(_=None):
    """The reference CPU path on K elements of config-3 layer 0: its per-axis Lagrange fibre
    transforms (mvpoly.py:193-230 `_lagrange_1d`, the kernel of interpolate_lagrange
    233-247) over fibres worth K elements on every axis, then the commitment MSM over K
    coefficients with K SRS points as the reference composes it (fold of
    PairingBackend.exp + mul, backend.py:185-217).  Returns seconds."""
    fns, fibres, coeffs, bases, backend = _TASK
    t0 = time.perf_counter()
    for j, fib in fibres:
        for f in fib:
            fns[j](f)
    if backend is not None:
        acc = None
        for a, b in zip(coeffs, bases):
            acc = backend.mul(acc, backend.exp(b, a))
    else:
        from oracle import tc_oracle as O
        O.msm_naive(coeffs, bases)
    return time.perf_counter() - t0


def cpu_sample(shape, K=48):
    """Inputs of the bounded CPU sample (one-time setup, untimed, no GPU): layer 0's
    quantised values cut into fibres of every axis worth K elements each, K interpolation
    coefficients (uniform F_p elements — what the 162-bit monomial coefficients of these
    activations look like; exp / mul time does not depend on which) and K curve points."""
    import random

    import numpy as np

    from oracle import tc_oracle as O
    backend_m, field_m, mvpoly_m, kind = _ref_modules()
    x = make_layers_host(CONFIGS[3], [0])[0].reshape(-1)
    q = O.quantize(x.astype(np.float64), 16)
    fibres, fns = [], []
    for j, d in enumerate(shape):
        stride = int(np.prod(shape[j + 1:]))
        fib = [[q[(f * stride * d + r * stride) % len(q)] for r in range(d)] for f in range(max(1, K // d))]
        fibres.append((j, fib))
        if mvpoly_m is not None:
            dom = field_m.PrimeField(backend_m.make_backend("production").order)
            fns.append(mvpoly_m._lagrange_1d(dom, list(range(1, d + 1))))
        else:
            rows = O.lagrange_matrix(list(range(1, d + 1)))
            fns.append(lambda fib, rows=rows, d=d: [sum(v * rows[l][k] for l, v in enumerate(fib)) % O.P
                                                    for k in range(d)])
    rng = random.Random(2602)
    coeffs = [rng.randrange(O.P) for _ in range(K)]
    bases = [O.ec_mul(O.G, k + 2) for k in range(K)]
    backend = backend_m.make_backend("production") if backend_m is not None else None
    return (fns, fibres, coeffs, bases, backend), K, kind


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_reference(shape, cores, target_s=8.0, single_s=2.0):
    """Throughput (elems/s) of the reference CPU path: one process (single-core figure) and
    `cores` processes (all host cores), each sized to ~target_s of wall time."""
    import multiprocessing as mp
    global _TASK
    _TASK, K, kind = cpu_sample(shape)
    one = _cpu_task()                                       # calibration (untimed)
    n1 = max(1, int(single_s / max(one, 1e-3)))
    t0 = time.perf_counter()
    for _ in range(n1):
        _cpu_task()
    single = K * n1 / (time.perf_counter() - t0)
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_cpu_task, range(cores))                   # warm the workers (untimed)
        rounds = max(1, int(target_s / max(one, 1e-3)))
        t0 = time.perf_counter()
        pool.map(_cpu_task, range(cores * rounds))
        wall = time.perf_counter() - t0
    n_tasks = cores * rounds
    return {"value": K * n_tasks / wall, "single_core": single, "wall_s": wall, "tasks": n_tasks, "K": K,
            "kind": kind}


def _cpu_line(cpu, cores):
    src = ("the unmodified reference modules (oracle/_ref, copied from the reference by oracle/make_ref.py): "
           "mvpoly._lagrange_1d fibre transforms + PairingBackend.exp/mul fold" if cpu["kind"] == "reference" else
           "the oracle's CPython restatement of the reference path (oracle/_ref absent)")
    return {"value": cpu["value"], "unit": "elems/s", "cores": cores, "kind": cpu["kind"],
            "single_core_value": cpu["single_core"], "cpu_model": cpu_model(),
            "sample": f"{cpu['tasks']} tasks x {cpu['K']} elements of config-3 layer 0 on {cores} processes "
                      f"({cpu['wall_s']:.1f} s): per-axis Lagrange fibre transforms worth those elements on every "
                      f"axis + naive MSM over K coefficients; {src}; extrapolated linearly per element"}


# ------------------------------------------------------------------ launch
def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reexec_torchrun(args):
    """bench.py --gpus N outside torchrun: relaunch as N ranks (one process per GPU)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator lines (NVLink / NVLS) in stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[3, 4, 5])
    ap.add_argument("--route", default="lagrange", choices=["lagrange", "monomial"])
    ap.add_argument("--no-forward", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-monomial", action="store_true", help="skip the secondary monomial-route step")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_reexec_torchrun(args))

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # TC_DIST_BACKEND=gloo lets several ranks share one GPU in tests (the kernels of the ranks
    # never wait on one another; the gather goes through host memory)
    backend = os.environ.get("TC_DIST_BACKEND", "nccl")
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    cfg = CONFIGS[5 if args.config == 5 else 3]

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg, cores, world)
        return    # other ranks: no work (no process group needed)

    dev_index = local if backend == "nccl" else local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", dev_index)
    try:
        if args.config == 4:
            run_openings(args, dev, rank, world, cores)
        else:
            run_commits(args, cfg, dev, rank, world, cores, backend)
    finally:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()


def _max_over_ranks(ms, world, dev, backend):
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_commits(args, cfg, dev, rank, world, cores, backend):
    import torch
    import torch.distributed as dist

    import paper_2602_12630_b200 as tcb
    from paper_2602_12630_b200 import _lib
    from paper_2602_12630_b200.dist import prover_commit_pipeline_dist, work_partition

    local = dev.index
    n_layers = cfg["layers"]
    shape = cfg["shape"]
    elems_per_layer = int(__import__("numpy").prod(cfg["act"]))
    per_step_elems = n_layers * elems_per_layer
    parts = work_partition(n_layers, elems_per_layer, world)[rank]
    my_layers = sorted({l for l, _, _ in parts})
    if args.config == 5:
        dev_layers = make_layers_device(cfg, my_layers, dev)
        host_pinned = [d.cpu().pin_memory() for d in dev_layers]
    else:
        host_pinned = [torch.from_numpy(h).pin_memory() for h in make_layers_host(cfg, my_layers)]
        dev_layers = [h.to(dev) for h in host_pinned]
    torch.cuda.synchronize(dev)
    # ---- setup (trusted setup, tables): timed and declared, outside the measured steps
    t0 = time.perf_counter()
    srs, _ = tcb.setup_srs(shape, b"tc-b200/config%d" % (5 if args.config == 5 else 3), device=local)
    torch.cuda.synchronize(dev)
    setup_ms = 1e3 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    srs.prepare("float16")
    torch.cuda.synchronize(dev)
    exptab_ms = 1e3 * (time.perf_counter() - t0)
    tcfg = tcb.TreeConfig(shape=NODE_SHAPE)
    node_srs = tcb.authtree.node_srs(tcfg, device=local)
    ctx = _lib.Context.get(local)
    PIPE_DEPTH = int(os.environ.get("TC_PIPE_DEPTH", "4"))
    use_pipe = not os.environ.get("TC_BENCH_NO_PIPELINE")
    dev_fwd = dict(zip(my_layers, dev_layers))
    host_fwd = dict(zip(my_layers, host_pinned))
    host_pinned2 = [h.clone().pin_memory() for h in host_pinned]   # "the next forward"
    host_fwd2 = dict(zip(my_layers, host_pinned2))

    def forwards(steps, host=False):
        if host:
            return [host_fwd if k % 2 == 0 else host_fwd2 for k in range(steps)]
        return [dev_fwd] * steps

    def run(steps, route=args.route, host=False):
        """`steps` forwards; every forward's commitments, root and tree read back."""
        root = None
        if world > 1:
            # per rank: its share of the (layer, element) space through the forward pipeline;
            # part encodings all-gathered on the device (NCCL), tree built on every rank
            for _, root, _ in prover_commit_pipeline_dist(forwards(steps, host), srs, n_layers, rank, world,
                                                          tree_config=tcfg, node_srs=node_srs, route=route,
                                                          depth=PIPE_DEPTH):
                pass
            return root
        if host and args.config == 5:
            # config 5: one context, forward k+1's upload under forward k's commitments
            batches = [host_pinned if k % 2 == 0 else host_pinned2 for k in range(steps)]
            for _, root, _ in tcb.prover_commit_stream(batches, srs, tree_config=tcfg, node_srs=node_srs,
                                                       route=route):
                pass
            return root
        if use_pipe:
            fw = [[f[l] for l in my_layers] for f in forwards(steps, host)]
            for _, root, _ in tcb.prover_commit_pipeline(fw, srs, tree_config=tcfg, node_srs=node_srs, route=route,
                                                         depth=PIPE_DEPTH):
                pass
            return root
        for f in forwards(steps, host):
            root = tcb.prover_commit([f[l] for l in my_layers], srs, tree_config=tcfg, node_srs=node_srs,
                                     route=route)[1]
        return root

    def all_launches():
        return ctx.launches + sum(c.launches for c in _lib.Context._pipeline.values())

    def timed(fn):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = all_launches()
        e0.record()
        root = fn()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = _max_over_ranks(e0.elapsed_time(e1), world, dev, backend)
        return ms, all_launches() - l0, root

    run(max(args.warmup, PIPE_DEPTH))                     # warm every pipeline context
    with Clocks(local) as clk:
        ms, launches, root = timed(lambda: run(args.steps))
    run(max(2, min(args.warmup, PIPE_DEPTH)), host=True)
    ms_e2e, _, root_e2e = timed(lambda: run(args.steps, host=True))
    if root_e2e != root:
        raise RuntimeError("e2e root differs from the device-resident root")
    # latency of ONE forward (nothing else in flight): the lone prover_commit
    lat = []
    for _ in range(3):
        lat.append(timed(lambda: run(1))[0])
    latency_ms = min(lat)

    # dominant kernel: Pippenger bucket accumulation, CUDA events on the ctx stream
    ctx.set_profiling(True)
    tcb.prover_commit([dev_fwd[l] for l in my_layers], srs, tree_config=tcfg, node_srs=node_srs)
    st = ctx.kernel_stats("msm.accumulate")
    ctx.set_profiling(False)
    import ctypes
    peak = ctypes.c_double()
    ctx.check(_lib.lib().tc_measure_imad_peak(ctx.handle, ctypes.byref(peak)))
    peak_tops = peak.value

    # trapdoor-free setup path: Lagrange elements derived from a monomial-only SRS
    derive_ms = None
    if rank == 0:
        mono_srs, _ = tcb.setup_srs(shape, b"tc-b200/derive", lagrange=False, device=local)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        mono_srs.derive_lagrange()
        torch.cuda.synchronize(dev)
        derive_ms = 1e3 * (time.perf_counter() - t0)
        del mono_srs

    # secondary: the monomial route (interpolate -> 162-bit-scalar MSM, SPEC.md:279 verbatim)
    mono = None
    if not args.no_monomial and args.route == "lagrange" and args.config == 3 and world == 1:
        run(1, route="monomial")
        m_ms, _, m_root = timed(lambda: run(1, route="monomial"))
        if m_root != root:
            raise RuntimeError("monomial route root differs from the Lagrange route")
        mono = {"ms_per_step": m_ms, "elems_per_s": per_step_elems / (m_ms / 1e3), "root_equal": True}

    ms_step = ms / args.steps
    value = per_step_elems / (ms_step / 1e3)
    achieved = st["units"] * WORD_MULS_PER_ADD / (st["ms"] * 1e-3) / 1e12 if st["ms"] else None
    traffic = None   # dram bytes per launch of k_accum_aff from the committed ncu --set full capture
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_accum_summary.txt")) as fh:
            kv = dict(l.split(" = ", 1) for l in fh if " = " in l)
        to_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic = sum(float(kv[k].split()[0]) * to_b[kv[k].split()[1]]
                      for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except (OSError, KeyError, ValueError, IndexError):
        pass

    fwd = None if (args.no_forward or rank != 0 or args.config != 3) else forward_ms(dev)
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = _cpu_line(cpu_reference(CONFIGS[3]["shape"], cores), cores)
    h2d = sum(t.numel() * t.element_size() for t in host_pinned)
    tree_d2h = (n_layers + 9) * 48 + 72 * 24     # commitments + node points (48-B affine), level values
    e2e = {"value": per_step_elems / (ms_e2e / args.steps / 1e3), "unit": "elems/s",
           "ms_per_step": ms_e2e / args.steps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": tree_d2h,
           "path": (f"{args.steps} forwards of pinned host tensors through the public API: "
                    + ("dist.prover_commit_pipeline_dist per rank (its share uploaded on a pipeline context's "
                       "stream, committed, part encodings all-gathered on the device, tree on every rank)"
                       if world > 1 else
                       "protocol.prover_commit_stream (one context; forward k+1's upload under forward k's "
                       "commitments)" if args.config == 5 else
                       f"protocol.prover_commit_pipeline ({PIPE_DEPTH} device contexts in turn: each uploads its "
                       "forward on its own copy stream and commits it while the others' forwards compute)")
                    + "; commitments, root and tree read back every forward; first upload exposed")}
    tables = srs.table_bytes()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elems/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32 (6-limb F_p/F_q Montgomery); input fp16", "data": "synthetic",
            "config": {"workload": cfg["name"], "route": args.route, "elems_per_step": per_step_elems,
                       "parallelism": f"layers/{world}" if all(c == elems_per_layer for _, _, c in parts)
                       else f"layer-chunks/{world}",
                       "l2": "no flush: fp16 inputs (>=128 MiB) + SRS (>=96 MiB) exceed the 126 MB L2",
                       "srs": "generated once before timing (trusted setup)",
                       "setup_ms": setup_ms, "exptab_build_ms": exptab_ms,
                       "lagrange_derive_ms": derive_ms, **tables,
                       "step_api": ("dist.prover_commit_pipeline_dist" if world > 1 else
                                    f"protocol.prover_commit_pipeline over the {args.steps} timed forwards "
                                    f"({PIPE_DEPTH} contexts; every forward's commitments, root and tree read back)"
                                    if use_pipe else "protocol.prover_commit per forward")},
            "latency_ms": latency_ms,
            "overhead_pct": (100.0 * ms_step / fwd) if fwd else None,
            "overhead_pct_ideal": 100.0 * ms_step / IDEAL_FORWARD_MS if args.config == 3 else None,
            "latency_overhead_pct_ideal": 100.0 * latency_ms / IDEAL_FORWARD_MS if args.config == 3 else None,
            "forward_ms": fwd, "forward_ms_ideal": IDEAL_FORWARD_MS,
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "int", "kernel": "k_accum_aff (Pippenger bucket accumulation)",
                         "achieved": achieved, "peak": peak_tops, "unit": "T word-mul/s",
                         "frac": (achieved / peak_tops) if achieved and peak_tops else None, "traffic": traffic,
                         "traffic_note": "dram read+write bytes per launch of the same kernel on the same workload "
                                         "(profiles/r02_ncu_accum_summary.txt)",
                         "work": f"{st['units']:.0f} bucket entries x {WORD_MULS_PER_ADD} word-muls "
                                 f"(11 mulmods x 78) over {st['launches']} launches, {st['ms']:.3f} ms",
                         "work_note": "counted per EXECUTED bucket add (one per element on the Lagrange route: the "
                                      "exponent table 2^g G_i, built at setup, absorbs the scalar's exponent)",
                         "peak_source": "mad.lo.u32 microbenchmark in this run (tc_measure_imad_peak)",
                         "share_of_step": st["ms"] / ms_step if ms_step else None},
            "monomial_route": mono,
            "cpu_baseline": cpu,
            "route_matched": ({"monomial_route_vs_cpu": mono["elems_per_s"] / cpu["value"],
                               "lagrange_route_vs_cpu": value / cpu["value"],
                               "note": "the CPU arm runs the reference's monomial path (interpolate + 162-bit MSM); "
                                       "the GPU monomial route is the same algorithm"}
                              if mono and cpu else None),
            "clocks": clk.summary(),
            "root": root.to_bytes().hex(),
        }
        print(json.dumps(line), flush=True)


IDEAL_FORWARD_MS = 4.87   # LLaMA-2-7B [1,512] forward: 6.83 TFLOP at the measured 1403.6 TFLOP/s


def run_reference(args, cfg, cores, world):
    """The reference arm: the reference's own CPU path (oracle/_ref) on all host cores, each
    step a bounded sample of the workload."""
    global _TASK
    _TASK, K, kind = cpu_sample(CONFIGS[3]["shape"])
    import multiprocessing as mp
    one = _cpu_task()
    # each step a bounded sample: ~6 s, less for long runs (the whole run stays ~2 minutes)
    per_step_s = min(6.0, max(1.0, 120.0 / max(1, args.steps)))
    rounds = max(1, int(per_step_s / max(one, 1e-3)))
    walls, tasks = [], 0
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(max(1, args.warmup)):
            pool.map(_cpu_task, range(cores))
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_cpu_task, range(cores * rounds))
            walls.append(time.perf_counter() - t0)
            tasks += cores * rounds
    value = tasks * K / sum(walls)
    cpu = _cpu_line({"value": value, "single_core": None, "wall_s": sum(walls), "tasks": tasks, "K": K, "kind": kind},
                    cores)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "elems/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int (CPython big int)",
            "data": "synthetic", "config": {"workload": cfg["name"], "parallelism": f"cpu x{cores}"},
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "elems/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config4_challenges(n_layers, shape, P):
    """256 seeded challenges spread over layers by a heavy-tailed (Pareto) score vector."""
    import random

    import numpy as np
    score = np.random.default_rng(4).pareto(1.5, n_layers) + 1e-3
    picks = np.random.default_rng(5).choice(n_layers, size=256, p=score / score.sum())
    rng = random.Random(6)
    return [(int(l), [rng.randrange(P) for _ in shape]) for l in picks]


def run_openings(args, dev, rank, world, cores):
    """Config 4: batched opening proofs on the config-3 tree — 256 seeded challenges spread
    over layers by a heavy-tailed score vector; each is tc_open (quotients + MSM) plus a
    Terkle membership proof.  N > 1: the challenges split over the ranks by cost
    (dist.open_many_dist), every proof gathered to every rank.  Reports openings/s
    (correctness: tests/test_gpu_fullsize.py checks every opening with the oracle verifier)."""
    import torch
    import torch.distributed as dist

    import paper_2602_12630_b200 as tcb
    from paper_2602_12630_b200.dist import hot_layer_plan, open_many_dist, prover_commit_dist, work_partition
    cfg = CONFIGS[3]
    n_layers = cfg["layers"]
    chals = config4_challenges(n_layers, cfg["shape"], tcb.P)
    hot, _, assign = hot_layer_plan([l for l, _ in chals], world, cfg["shape"][0], len(cfg["shape"]))
    mine = assign[rank] if world > 1 else list(range(len(chals)))
    n_elems = int(__import__("numpy").prod(cfg["act"]))
    # this rank's challenged layers, the hot layers (every rank computes rows of their slice
    # commitments) and the layers of its commitment share (dist.py)
    need = sorted({chals[i][0] for i in mine} | (set(hot) if world > 1 else set())
                  | {l for l, _, _ in work_partition(n_layers, n_elems, world)[rank]})
    host = dict(zip(need, make_layers_host(cfg, need)))
    layers = {l: torch.from_numpy(h).to(dev) for l, h in host.items()}
    srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/config3", device=dev.index)
    srs.prepare("float16")
    if world > 1:
        comms, root, tree = prover_commit_dist(layers, srs, n_layers, rank, world)
    else:
        comms, root, tree = tcb.prover_commit([layers[l] for l in range(n_layers)], srs, return_tree=True)

    def step(tr):
        return open_many_dist(srs, layers, chals, rank, world, tree=tr)

    for _ in range(max(1, args.warmup)):       # window tables, slice / table-kernel paths
        step(tcb.build(tree.config, tree.values[0][:tree.n], srs=tree.srs)[0])
    fresh = tcb.build(tree.config, tree.values[0][:tree.n], srs=tree.srs)[0]   # no memoised node openings
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops, proofs = step(fresh)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = _max_over_ranks(e0.elapsed_time(e1), world, dev, os.environ.get("TC_DIST_BACKEND", "nccl"))
    # spot-check: openings verify on the CPU verifier, membership proofs too (the full check
    # of all 256 with the oracle verifier is tests/test_gpu_fullsize.py)
    for k in (0, len(chals) // 2, len(chals) - 1):
        l, pt = chals[k]
        if not tcb.tc_verify(srs, comms[l], pt, ops[k]):
            raise RuntimeError("config-4 opening does not verify")
        if not tcb.verify(root, l, tcb.authtree.leaf_of(comms[l]), proofs[k], tree.config):
            raise RuntimeError("config-4 membership proof does not verify")
    if rank == 0:
        print(json.dumps({"metric": "opening proofs/sec (tc_open + Terkle membership proof)",
                          "value": len(chals) / (ms / 1e3), "unit": "openings/s", "n_gpus": world,
                          "ms_per_opening": ms / len(chals), "ms_total": ms, "higher_is_better": True,
                          "config": {"workload": "config4: 256 challenges on the config-3 tree, layers drawn by a "
                                                 "seeded Pareto score vector, random field points",
                                     "parallelism": f"openings/{world} (hot layers' slice commitments split by rows over "
                                                    "the ranks + one all-gather; openings dealt out by cost)",
                                     "path": "dist.open_many_dist -> tc_open_slices (rank's rows of H[c',c]) + all-gather "
                                             "+ tc_open_batch_sliced (pi_0 as a d0^2-point MSM over H) for layers opened "
                                             ">= 6 times, tc_open_many (grouped quotient MSMs) for the others; "
                                             "prove_many (node openings batched)"}}),
              flush=True)


if __name__ == "__main__":
    main()
