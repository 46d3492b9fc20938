#!/usr/bin/env python
"""Benchmark of the COMM-RAND mini-batch hot path on B200 (BASELINE.json metric).

A step = one pass of the whole hot path over one mini-batch of the
products-shaped synthetic workload (BASELINE.json configs[3]; the config the
metric's "1/2/4/8 B200" is quoted on): Knob-2 biased 3-hop sampling + dedup/
relabel (a2, a3) and the fused input-feature gather + GraphSAGE-mean aggregation
(a4, a5); the Knob-1 root order (a1) is recomputed at the start of the timed
region and at every epoch boundary inside it (it is once per epoch).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cmb|reference]
                  [--config products|papers100m|...] [--shard none|ipc|a2a]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

`--gpus N` without a torchrun environment re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL).

Multi-GPU: batches are independent units (reading R22): rank r runs global
batches r, r+N, r+2N, ... with the graph and features replicated; there is no
per-batch collective (weak scaling).  `--shard ipc|a2a` row-shards the feature table
over the ranks instead (a6, the papers100M layout of BASELINE.json configs[4]): `ipc` reads
remote rows inside the fused gather through CUDA-IPC-mapped peer shards (NEXT-1, NVLink on a
multi-GPU node), `a2a` exchanges ids and rows with NCCL all-to-all (shard.ShardedFeatures).
Rank 0 prints one JSON line.
"""
from __future__ import annotations

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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="cmb", choices=["cmb", "reference"])
    ap.add_argument("--config", default="products")
    ap.add_argument("--mode", default="rand", choices=["rand", "norand", "comm", "comm_static"])
    ap.add_argument("--mix", type=float, default=0.0)
    ap.add_argument("--p", type=float, default=None)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--no-extra", action="store_true", help="skip the knob-sweep extra points")
    ap.add_argument("--layer", action="store_true",
                    help="with --no-extra: still measure the NEXT-4 fused layer point")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--law", default="A", choices=["A", "slot"],
                    help="Knob-2 law: A = weighted w/o replacement (default), slot = R23")
    ap.add_argument("--flush-l2", default="auto", choices=["auto", "on", "off"],
                    help="write 256 MB before every launch group and time only the groups "
                         "(auto: on when features + CSR < 4x L2)")
    ap.add_argument("--batches-per-launch", type=int, default=None,
                    help="batches sampled per persistent-sampler launch (1..8; default "
                         "cmb.DEFAULT_BATCHES_PER_LAUNCH = 6, measured best on products)")
    ap.add_argument("--shard", default="none", choices=["none", "ipc", "a2a"],
                    help="row-shard the feature table over the ranks (a6): ipc = one-sided "
                         "gather of peer shards mapped by CUDA IPC, a2a = NCCL all-to-all")
    ap.add_argument("--out-ld", type=int, default=0,
                    help="row stride (floats) of the X_in / H outputs; 0 = the feature table's "
                         "(layout experiments: a multiple of 8 starts every row on a 32-B sector)")
    ap.add_argument("--train-graph", default="on", choices=["on", "off"],
                    help="replay each NEXT-4 training step as a captured CUDA graph "
                         "(GraphSAGE.train_step(graph=True)) or enqueue it launch by launch")
    ap.add_argument("--dst-order", default="on", choices=["on", "off"],
                    help="let the sampler write the last hop's dst visiting order for the fused "
                         "gather (cmb_blocks.dst_order; same bytes either way) -- A/B switch")
    ap.add_argument("--cpu-workers", type=int, default=0,
                    help="threads of the batch-parallel oracle baseline (0 = all host cores)")
    args = ap.parse_args()
    if args.batches_per_launch is None:
        from paper_2504_18082_b200 import DEFAULT_BATCHES_PER_LAUNCH  # (no library load)
        args.batches_per_launch = DEFAULT_BATCHES_PER_LAUNCH
    return args


def relaunch(args):
    """`--gpus N` outside a torchrun environment: start N ranks (one per GPU) under
    torch.distributed.run on this node and return its exit status (rank 0 prints the line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def host_cpu():
    """(logical cores, CPU model) of this host."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count() or 1, model


METRIC = "mini-batches/s"


# ------------------------------------------------------------------ helpers
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every ~5 ms during the timed
    region through NVML (the same counters nvidia-smi's clocks line reads)."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.max_mhz = None
        self.error = None
        self._stop = threading.Event()
        self._t = None
        self._h = None
        try:  # NVML opened in the caller's thread; a failure is reported, not hidden
            import pynvml
            self._nv = pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.error = f"{type(e).__name__}: {e}"

    def _sample(self):
        try:
            sm = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
            rs = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.rows.append((sm, rs))
        except Exception as e:  # noqa: BLE001
            self.error = f"{type(e).__name__}: {e}"

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.005)

    def __enter__(self):
        if self._h is not None:
            self._sample()  # at least one sample per region, however short
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()
        if self._h is not None:
            self._sample()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"],
                    "error": self.error}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for _, rs in self.rows for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "NVML during the timed region"}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload, knob):
    """Per-launch DRAM bytes of the fused gather/aggregate kernel from the committed
    ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(f"{workload}|{knob}")
    except Exception:
        return None


def algorithmic_bytes(n, e, F, L):
    """Fused a4+a5 launch: every unique input row read once
    (U*R), X_in written (U*R), H written (n_{L-1}*R), plus the int32 index streams
    (indices of hop L-1, indptr of hop L-1, the relabel map nodes[0:U))."""
    R = 4 * F
    U, nd, ed = n[L], n[L - 1], e[L - 1]
    return 2 * U * R + nd * R + 4 * ed + 4 * (nd + 1) + 4 * U


# ------------------------------------------------------------------ cpu (oracle) legs
def oracle_step(prep, bundle, roots, p, seed, batch, scratch, law=0):
    """One oracle batch (a2-a5).  For device-generated feature tables the gathered rows come
    from the generator's row formula (X[nodes] by definition), then the oracle's a5."""
    import oracle
    from gen.planted import feature_rows
    cfg = bundle.cfg
    if bundle.X is not None:
        return oracle.run_batch(prep, bundle.X, cfg.feat_dim, roots, cfg.fanouts, p, seed, batch,
                                scratch, law)
    L = len(cfg.fanouts)
    blk = oracle.sample_blocks(prep, roots, cfg.fanouts, p, seed, batch, scratch, law)
    Xin = np.ascontiguousarray(feature_rows(bundle, blk["nodes"]))
    H, H64 = oracle.sage_mean(blk["indptr"][L - 1], blk["indices"][L - 1], Xin, cfg.feat_dim)
    blk.update({"X_in": Xin, "H": H, "H64": H64})
    return blk


def oracle_batches(bundle, mode, mix, p, seed, budget_s, max_batches=None, law=0):
    """Times the oracle (as it stands, single thread) on consecutive batches of epoch 0."""
    import oracle
    cfg = bundle.cfg
    prep = oracle.graph_prep(bundle)
    modes = {"rand": oracle.MODE_RAND, "norand": oracle.MODE_NORAND, "comm": oracle.MODE_COMM,
             "comm_static": oracle.MODE_COMM_STATIC}
    scratch = np.full(prep.num_nodes, -1, dtype=np.int32)
    t0 = time.perf_counter()
    order = oracle.order_roots(bundle.train, bundle.comm, cfg.num_communities, modes[mode], mix,
                               seed, 0)
    nb = (order.shape[0] + cfg.batch_size - 1) // cfg.batch_size
    done, edges = 0, 0
    while True:
        r = oracle_step(prep, bundle, oracle.batch_roots(order, cfg.batch_size, done % nb), p,
                        seed, done % nb, scratch, law)
        edges += sum(r["e"])
        done += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (max_batches and done >= max_batches):
            break
    return done, el, edges


def oracle_parallel(bundle, mode, mix, p, seed, n_batches=None, budget_s=None, workers=0, law=0,
                    first=0):
    """Batch-parallel oracle (SURVEY.md §8(d) mode 2): consecutive batches of epoch 0 run by a
    pool of `workers` threads, each batch the same plain single-threaded C functions (they
    release the GIL; batches are independent by reading R11).  Stops after `n_batches`, or once
    `budget_s` of wall time has passed.  Returns (batches, seconds, edges, threads)."""
    from concurrent.futures import FIRST_COMPLETED, ThreadPoolExecutor, wait
    import oracle
    cfg = bundle.cfg
    workers = workers or (os.cpu_count() or 1)
    prep = oracle.graph_prep(bundle)
    modes = {"rand": oracle.MODE_RAND, "norand": oracle.MODE_NORAND, "comm": oracle.MODE_COMM,
             "comm_static": oracle.MODE_COMM_STATIC}
    t0 = time.perf_counter()
    order = oracle.order_roots(bundle.train, bundle.comm, cfg.num_communities, modes[mode], mix,
                               seed, 0)
    nb = (order.shape[0] + cfg.batch_size - 1) // cfg.batch_size
    scratch = [np.full(prep.num_nodes, -1, dtype=np.int32) for _ in range(workers)]
    free = list(range(workers))

    def one(b):
        slot = free.pop()
        try:
            r = oracle_step(prep, bundle, oracle.batch_roots(order, cfg.batch_size, b % nb), p,
                            seed, b % nb, scratch[slot], law)
            return sum(r["e"])
        finally:
            free.append(slot)

    done = edges = 0
    nxt = first
    with ThreadPoolExecutor(max_workers=workers) as ex:
        live = set()
        while True:
            stop = (n_batches is not None and nxt - first >= n_batches) or \
                   (budget_s is not None and time.perf_counter() - t0 >= budget_s)
            while not stop and len(live) < workers:
                live.add(ex.submit(one, nxt))
                nxt += 1
                stop = n_batches is not None and nxt - first >= n_batches
            if not live:
                break
            fin, live = wait(live, return_when=FIRST_COMPLETED)
            for f in fin:
                edges += f.result()
                done += 1
            if stop and not live:
                break
    return done, time.perf_counter() - t0, edges, workers


def run_reference(args, bundle):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = bundle.cfg
    p = cfg.p_intra if args.p is None else args.p
    import oracle
    prep = oracle.graph_prep(bundle)
    modes = {"rand": oracle.MODE_RAND, "norand": oracle.MODE_NORAND, "comm": oracle.MODE_COMM,
             "comm_static": oracle.MODE_COMM_STATIC}
    order = oracle.order_roots(bundle.train, bundle.comm, cfg.num_communities, modes[args.mode],
                               args.mix, args.seed, 0)
    nb = (order.shape[0] + cfg.batch_size - 1) // cfg.batch_size
    scratch = np.full(prep.num_nodes, -1, dtype=np.int32)

    def step(b):
        return oracle_step(prep, bundle, oracle.batch_roots(order, cfg.batch_size, b % nb), p,
                           args.seed, b % nb, scratch, 0 if args.law == "A" else 1)

    for w in range(args.warmup):
        step(w)
    # the K timed steps (one batch each) run batch-parallel over the host's cores
    done, el, edges, workers = oracle_parallel(bundle, args.mode, args.mix, p, args.seed,
                                               n_batches=args.steps, workers=args.cpu_workers,
                                               law=0 if args.law == "A" else 1, first=args.warmup)
    cores, model = host_cpu()
    val = done / el
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "batches/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, cfg, bundle, p),
            "sampled_edges_per_s": edges / el,
            "cpu_baseline": {"value": val, "unit": "batches/s", "cores": workers, "kind": "oracle",
                             "host_cores": cores, "cpu_model": model,
                             "sample": f"{args.steps} consecutive batches of epoch 0 (one per "
                                       f"step), batch-parallel over {workers} threads, each batch "
                                       f"the single-threaded plain-C oracle (oracle/oracle.c), "
                                       f"a1 included"},
            "e2e": {"value": val, "unit": "batches/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


L2_BYTES = 126 << 20


def inputs_exceed_l2(cfg, bundle):
    return cfg.num_nodes * cfg.feat_ld * 4 + bundle.nnz * 4 > 4 * L2_BYTES


def workload_config(args, cfg, bundle, p, flush=False):
    return {"workload": f"{cfg.name}-shaped synthetic (BASELINE.json configs[3])"
            if cfg.name == "products" else f"{cfg.name}-shaped synthetic",
            "num_nodes": cfg.num_nodes, "nnz": int(bundle.nnz), "feat_dim": cfg.feat_dim,
            "batch": cfg.batch_size, "fanouts_hop_order": list(cfg.fanouts),
            "knob1": args.mode + (f"(k={args.mix})" if args.mode.startswith("comm") else ""),
            "dst_order": args.dst_order,
            "p_intra": p, "knob2_law": args.law, "seed": args.seed,
            "l2": ("L2 flushed (256 MB write) before every launch group of %d batches; "
                   "ms = sum of the groups' device events (X %.0f MB, CSR %.0f MB)"
                   % (args.batches_per_launch, cfg.num_nodes * cfg.feat_ld * 4 / 1e6,
                      bundle.nnz * 4 / 1e6)) if flush else
                  "no flush: inputs larger than L2 (X %.0f MB, CSR %.0f MB > 126 MB)"
                  % (cfg.num_nodes * cfg.feat_ld * 4 / 1e6, bundle.nnz * 4 / 1e6),
            "parallelism": (f"dp{int(os.environ.get('WORLD_SIZE', '1'))} (batches round-robin over "
                            f"ranks, graph replicated" +
                            (", features replicated)" if args.shard == "none" else
                             f", feature rows sharded over the ranks, {args.shard} exchange)"))}


# ------------------------------------------------------------------ gpu leg
def count_launches(fn):
    """Kernels our library launches in one call of fn (CUPTI via torch.profiler)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    ours = [n for n in names if ("cmb" in n or "cub" in n.lower()) and "emcpy" not in n and "emset" not in n]
    return len(ours), sorted(set(ours))


def init_ranks():
    """One process per GPU (torchrun environment, else a single rank): (world, rank, local,
    backend, device).  CMB_DIST_BACKEND=gloo (+ more ranks than GPUs) only to exercise the
    multi-rank flow on a single-GPU box."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("CMB_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return world, rank, local, backend, dev


def run_cmb(args, bundle):
    import torch
    import torch.distributed as dist
    import paper_2504_18082_b200 as cmb
    from paper_2504_18082_b200 import dist as cmb_dist

    world, rank, local, backend, dev = init_ranks()
    cfg = bundle.cfg
    p = cfg.p_intra if args.p is None else args.p
    L = len(cfg.fanouts)
    from gen.device import feature_table
    graph = cmb.Graph.from_bundle(bundle, device=dev, validate=True,
                                  features=feature_table(bundle, dev))
    G = max(1, min(args.batches_per_launch, cmb.MAX_BATCHES_PER_LAUNCH))
    pipe = cmb.BatchedPipeline(graph, torch.from_numpy(bundle.train), cfg.batch_size,
                               cfg.fanouts, mode=args.mode, mix=args.mix, p=p, seed=args.seed,
                               nb=G, law=args.law)
    for smp in pipe.samplers:
        smp.set_dst_order(args.dst_order == "on")
        if args.out_ld:
            smp.alloc_features_ld(args.out_ld)
    nb = pipe.n_batches
    stream = torch.cuda.current_stream()
    K, W = args.steps, args.warmup
    sizes_log = torch.zeros(K, 2 * L + 1, dtype=torch.int64, device=dev)

    def gbatch(t):  # global batch id of this rank's t-th step (round-robin, reading R22)
        return cmb_dist.global_batch(rank, world, t)

    def group(t0, count, events=None, sizes_out=None):
        """Steps t0 .. t0+count-1 of this rank: one sampler launch + one gather launch."""
        return pipe.step_group([gbatch(t) for t in range(t0, t0 + count)], events=events,
                               sizes_out=sizes_out)

    # warm-up (also compiles nothing: the library is prebuilt)
    for t in range(0, W, G):
        group(t, min(G, W - t))
    torch.cuda.synchronize()
    for obj in [graph, pipe.orderer] + list(pipe.samplers):
        st = obj.status()
        if st != 0:
            raise RuntimeError(f"device status {st} after warm-up")
    n_launch_group, kernel_names = count_launches(lambda: group(W, G))
    n_launch_order, _ = count_launches(lambda: pipe.start_epoch(pipe.epoch))

    flush = args.flush_l2 == "on" or (args.flush_l2 == "auto" and not inputs_exceed_l2(cfg, bundle))
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    evlog = []
    # per-group timing events created before the region (creating them inside costs host time)
    evpool = [pipe.make_events(min(G, K - k0)) for k0 in range(0, K, G)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    orders_in_region = 0
    n_groups = 0
    with ClockSampler(local) as clk:
        start.record(stream)
        pipe.start_epoch(gbatch(W) // nb)       # a1 for the current epoch, inside the region
        orders_in_region += 1
        for k0 in range(0, K, G):
            cnt = min(G, K - k0)
            ep0 = pipe.epoch
            orders_in_region += len({gbatch(W + k) // nb for k in range(k0, k0 + cnt)} - {ep0})
            evs = evpool[k0 // G]
            if flush:
                scrub.fill_(k0 & 0xFF)   # evicts the previous group's lines from L2
            ss = group(W + k0, cnt, evs, sizes_log[k0:k0 + cnt])  # sizes written in place
            evlog.append({"sample": (evs[0], evs[1]),
                          "gather": [(evs[2 + 2 * i], evs[3 + 2 * i]) for i in range(cnt)]})
            n_groups += 1
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end)
    if flush:  # the timed work is the groups themselves (first sampler start -> last gather end)
        ms = sum(ev["sample"][0].elapsed_time(ev["gather"][-1][1]) for ev in evlog)
    agg_ms = [g0.elapsed_time(g1) for ev in evlog for (g0, g1) in ev["gather"]]
    samp_ms = [ev["sample"][0].elapsed_time(ev["sample"][1]) / len(ev["gather"]) for ev in evlog
               for _ in ev["gather"]]
    sz = sizes_log.cpu().numpy()
    n_h = sz[:, : L + 1]
    e_h = sz[:, L + 1:]
    alg = [algorithmic_bytes(n_h[k], e_h[k], cfg.feat_dim, L) for k in range(K)]
    ms_max, (total_edges, total_batches) = cmb_dist.reduce_timing(
        ms, [float(e_h.sum()), float(K)], device=dev if backend == "nccl" else None)

    # ---------------- e2e: host buffers through the public API (rank-local)
    e2e = run_e2e(args, pipe, cfg, stream, K, W, world, rank)

    extra = None
    layer = None
    if not args.no_extra and world == 1:
        extra = knob_points(bundle, graph, cfg, args, K, flush)
    if (not args.no_extra or args.layer) and world == 1:
        layer = layer_point(bundle, graph, cfg, args)
        layer["train_step"] = train_point(bundle, graph, cfg, args)

    if rank == 0:
        peak, peak_src = measured_peak_hbm()
        achieved = float(np.mean(alg)) / (float(np.mean(agg_ms)) * 1e-3) / 1e9
        knob = args.mode + (f"(k={args.mix})" if args.mode.startswith("comm") else "") + f"|{p}"
        traffic = ncu_traffic(cfg.name, knob)
        cpu = None
        if world == 1:
            cpu = cpu_baseline(args, bundle, p)
        value = total_batches / (ms_max * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": "batches/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, cfg, bundle, p, flush),
            "sampled_edges_per_s": total_edges / (ms_max * 1e-3),
            "feature_gbps": achieved,
            "unique_input_rows_per_batch": float(n_h[:, L].mean()),
            "unique_feature_bytes_per_batch": float(n_h[:, L].mean() * 4 * cfg.feat_dim),
            "stage_ms_per_step": {"sample_relabel": float(np.mean(samp_ms)),
                                  "gather_aggregate": float(np.mean(agg_ms))},
            "roofline": {"bound": "hbm",
                         "kernel": "k_gather_mean_row (fused a4+a5, cmb_gather_aggregate)",
                         "achieved": achieved, "peak": peak, "peak_source": peak_src,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": float(np.mean(alg))},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(n_launch_group * n_groups + n_launch_order * orders_in_region),
            "gpu_launches_detail": {"per_group_of_batches": n_launch_group,
                                    "batches_per_sampler_launch": G, "groups": n_groups,
                                    "per_epoch_order": n_launch_order,
                                    "orders_in_region": orders_in_region,
                                    "kernels": kernel_names},
            "clocks": clk.summary(),
            "knob_points": extra,
            "knob_pearson_time_vs_feature_bytes": knob_pearson(extra, cfg) if extra else None,
            "next4_layer": layer,
            "graph_meta": {k: (float(v) if isinstance(v, (np.floating, float)) else v)
                           for k, v in bundle.meta.items()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_baseline(args, bundle, p):
    """§8(d): the oracle as it stands, timed on this host's cores on a bounded sample of the same
    workload -- batch-parallel over all cores (the headline `value`) and on one core."""
    law = 0 if args.law == "A" else 1
    d1, el1, _ = oracle_batches(bundle, args.mode, args.mix, p, args.seed, args.cpu_seconds / 3,
                                law=law)
    dn, eln, _, workers = oracle_parallel(bundle, args.mode, args.mix, p, args.seed,
                                          budget_s=args.cpu_seconds, workers=args.cpu_workers,
                                          law=law)
    cores, model = host_cpu()
    return {"value": dn / eln, "unit": "batches/s", "cores": workers, "kind": "oracle",
            "host_cores": cores, "cpu_model": model,
            "sample": f"first {dn} batches of epoch 0 of the same workload/knobs in {eln:.1f} s, "
                      f"batch-parallel over {workers} threads, each batch the single-threaded "
                      f"plain-C oracle (oracle/oracle.c), a1 included",
            "single_core": {"value": d1 / el1, "unit": "batches/s", "cores": 1,
                            "sample": f"first {d1} batches of epoch 0, one thread, {el1:.1f} s"}}


def run_sharded(args, bundle):
    """a6 / NEXT-1 at N ranks: the feature table row-sharded over the ranks (rank r owns rows
    [r*S, (r+1)*S), S = ceil(N / W), generated in place on its GPU), graph replicated.  Per launch
    group: one sampler launch for up to 4 batches, then per batch the input-feature gather +
    aggregate from the sharded table -- `ipc`: the fused kernel reading remote rows from the
    peers' shards mapped by CUDA IPC (cmb_gather_aggregate_sharded, no host sync, no staging);
    `a2a`: ids and rows exchanged with NCCL all-to-all (shard.ShardedFeatures; its variable
    splits need the counts on the host: one device->host read per batch, that arm's cost), then
    the unfused a5 over X_in.  A spot check against the generator's row formula follows."""
    import torch
    import torch.distributed as dist
    import paper_2504_18082_b200 as cmb
    from paper_2504_18082_b200 import dist as cmb_dist
    from paper_2504_18082_b200.shard import ShardedFeatures
    from gen.device import feature_table
    from gen.planted import feature_rows

    world, rank, local, backend, dev = init_ranks()
    cfg = bundle.cfg
    p = cfg.p_intra if args.p is None else args.p
    L, F, N, B = len(cfg.fanouts), cfg.feat_dim, cfg.num_nodes, cfg.batch_size
    S = (N + world - 1) // world
    r0, r1 = rank * S, min(N, (rank + 1) * S)
    x_local = feature_table(bundle, dev, r0, r1)
    graph = cmb.Graph.from_bundle(bundle, device=dev, validate=True, features=False)
    G = max(1, min(args.batches_per_launch, cmb.MAX_BATCHES_PER_LAUNCH))
    pipe = cmb.MiniBatchPipeline(graph, torch.from_numpy(bundle.train), B, cfg.fanouts,
                                 mode=args.mode, mix=args.mix, p=p, seed=args.seed, law=args.law)
    samplers = [pipe.sampler] + [cmb.Sampler(graph, B, cfg.fanouts) for _ in range(G - 1)]
    nb = pipe.n_batches
    if args.shard == "ipc":
        table = (cmb.ShardTable.exchange(x_local, N, F, rank, world) if world > 1 else
                 cmb.ShardTable([x_local], N, F))

        def gather(s):
            return s.gather_aggregate_sharded(table)
    else:
        sf = ShardedFeatures(x_local, N, F, world, rank)

        def gather(s):
            x_in, h = s.alloc_features_ld(x_local.stride(0))
            n = int(s.sizes[L].item())   # the a2a splits need host-side counts
            sf.gather(s.nodes, n, x_in)
            cmb.sage_mean_aggregate(s.indptr[L - 1], s.indices[L - 1], s.sizes[L - 1:L], x_in, F,
                                    h, n_dst_cap=s.n_cap[L - 1])
            return x_in, h

    def gbatch(t):
        return cmb_dist.global_batch(rank, world, t)

    def group(t0, cnt, ev=None):
        ids = [gbatch(t) for t in range(t0, t0 + cnt)]
        roots = []
        for gb in ids:
            e, bb = divmod(gb, nb)
            if pipe.epoch != e:
                roots = [r.clone() for r in roots]
                pipe.start_epoch(e)
            roots.append(pipe.batch_roots(bb))
        if ev:
            ev[0].record()
        cmb.sample_multi(samplers[:cnt], roots, ids, p, args.seed, args.law)
        if ev:
            ev[1].record()
        for i, s in enumerate(samplers[:cnt]):
            gather(s)
        if ev:
            ev[2].record()
        return samplers[:cnt]

    K, W = args.steps, args.warmup
    for t in range(0, W, G):
        group(t, min(G, W - t))
    torch.cuda.synchronize()
    sizes_log = torch.zeros(K, 2 * L + 1, dtype=torch.int64, device=dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(0, K, G)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record()
        for gi, k0 in enumerate(range(0, K, G)):
            cnt = min(G, K - k0)
            ss = group(W + k0, cnt, evs[gi])
            for i, s in enumerate(ss):
                sizes_log[k0 + i].copy_(s.sizes, non_blocking=True)
        end.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end)
    samp = sum(e[0].elapsed_time(e[1]) for e in evs) / K
    gat = sum(e[1].elapsed_time(e[2]) for e in evs) / K
    sz = sizes_log.cpu().numpy()
    n_h, e_h = sz[:, : L + 1], sz[:, L + 1:]
    alg = float(np.mean([algorithmic_bytes(n_h[k], e_h[k], F, L) for k in range(K)]))
    # remote share of the last batch's unique input rows (the rows read over NVLink / exchanged)
    s_last = ss[-1]
    nl = int(sz[K - 1, L])
    remote = cmb_dist.remote_fraction(s_last.nodes, nl, rank, S)
    # spot check against the generator's row formula (input generation, not the method): X_in
    # rows byte-identical to X[nodes], H rows = fp64 mean of their X_in rows within 1e-5
    rng = np.random.default_rng(rank)
    x_in, h = s_last.x_in, s_last.h
    nodes = s_last.nodes[:nl].cpu().numpy()
    pick = rng.choice(nl, size=min(nl, 2048), replace=False)
    ok_x = bool(np.array_equal(x_in[torch.from_numpy(pick).to(dev), :F].cpu().numpy(),
                               feature_rows(bundle, nodes[pick])))
    ip = s_last.indptr[L - 1][: int(sz[K - 1, L - 1]) + 1].cpu().numpy().astype(np.int64)
    ix = s_last.indices[L - 1][: int(sz[K - 1, L + 1 + L - 1])].cpu().numpy()
    rows = rng.choice(ip.shape[0] - 1, size=min(ip.shape[0] - 1, 256), replace=False)
    xin_h = x_in[: nl, :F].cpu().numpy()
    hh = h[: ip.shape[0] - 1, :F].cpu().numpy()
    ok_h = True
    for d in rows:
        a, b_ = ip[d], ip[d + 1]
        want = xin_h[ix[a:b_]].astype(np.float64).mean(0) if b_ > a else np.zeros(F)
        scale = np.abs(xin_h[ix[a:b_]]).astype(np.float64).mean(0) if b_ > a else np.zeros(F)
        ok_h &= bool(np.all(np.abs(hh[d] - want) <= 1e-5 * np.maximum(np.abs(want), scale) + 1e-30))
    ok = torch.tensor([int(ok_x and ok_h)], dtype=torch.int64, device=dev)
    ms_max, (tot_edges, tot_batches, n_ok) = cmb_dist.reduce_timing(
        ms, [float(e_h.sum()), float(K), float(ok.item())],
        device=dev if backend == "nccl" else None)
    if int(n_ok) != world:
        raise RuntimeError(f"sharded gather spot check failed on {world - int(n_ok)} rank(s)")
    if rank == 0:
        peak, peak_src = measured_peak_hbm()
        achieved = alg / (gat * 1e-3) / 1e9
        remote_bytes = remote * float(np.mean(n_h[:, L])) * 4 * F
        line = {
            "metric": METRIC, "value": tot_batches / (ms_max * 1e-3), "unit": "batches/s",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_max / K,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": workload_config(args, cfg, bundle, p),
            "sampled_edges_per_s": tot_edges / (ms_max * 1e-3),
            "stage_ms_per_step": {"sample_relabel": samp, "gather_aggregate_sharded": gat},
            "unique_input_rows_per_batch": float(n_h[:, L].mean()),
            "roofline": {"bound": "hbm" if world == 1 else "nvlink",
                         "kernel": ("k_gather_mean_row<ShardedRows> (cmb_gather_aggregate_sharded)"
                                    if args.shard == "ipc" else
                                    "NCCL all-to-all exchange + k_gather_v4 / k_scatter_rows + "
                                    "k_gather_mean_pipe"),
                         "achieved": achieved, "peak": peak, "peak_source": peak_src,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                         "algorithmic_bytes_per_launch": alg},
            "nvlink": {"remote_row_fraction": remote,
                       "remote_bytes_per_batch": remote_bytes,
                       "remote_gbps": remote_bytes / (gat * 1e-3) / 1e9,
                       "peak_gbps_per_direction_spec": 900.0,
                       "note": "ranks on distinct GPUs read remote rows over NVLink; ranks that "
                               "share one GPU (a functional dry run) read them from the same HBM"},
            "spot_check": {"x_in_rows": int(pick.shape[0]), "h_rows": int(rows.shape[0]),
                           "ok_all_ranks": True},
            "cpu_baseline": None, "e2e": None,
            "gpu_launches": None,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if args.shard == "ipc" and world > 1:
        table.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_e2e(args, pipe, cfg, stream, K, W, world, rank):
    """Same metric through the public API with HOST buffers: per step the batch's roots
    are copied host->device from pinned memory and the batch's result sizes
    (n_0..n_L, e_0..e_{L-1}) are read back device->host and consumed by the host."""
    import torch
    L = len(cfg.fanouts)
    nb = pipe.n_batches
    G = pipe.nb
    dev = pipe.sampler.sizes.device
    B = cfg.batch_size
    order_host = torch.empty(pipe.orderer.n, dtype=torch.int32, pin_memory=True)
    # two slots: the host enqueues launch group k+1 while the device runs group k, then waits for
    # group k's sizes only (one group in flight, the way a training loop overlaps its data path)
    roots_dev = [[torch.empty(B, dtype=torch.int32, device=dev) for _ in range(G)] for _ in range(2)]
    sizes_host = [torch.empty(G, 2 * L + 1, dtype=torch.int64, pin_memory=True) for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    h2d = d2h = 0
    epoch_cache = {}

    def enqueue(t0, count, slot):
        """Steps t0 .. t0+count-1 (one sampler launch): per batch a pinned H2D copy of its
        roots, the step, then a D2H copy of its sizes into the slot; returns the count."""
        nonlocal h2d, d2h
        gbs = [t * world + rank for t in range(t0, t0 + count)]
        roots = []
        for i, gb in enumerate(gbs):
            epoch, b = divmod(gb, nb)
            if epoch_cache.get("epoch") != epoch:
                pipe.start_epoch(epoch)
                order_host.copy_(pipe.order, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                epoch_cache["epoch"] = epoch
                d2h += order_host.numel() * 4
            lo, hi = b * B, min((b + 1) * B, pipe.orderer.n)
            r = roots_dev[slot][i][: hi - lo]
            r.copy_(order_host[lo:hi], non_blocking=True)
            h2d += (hi - lo) * 4
            roots.append(r)
        pipe.step_group(gbs, roots=roots)
        sizes_host[slot][:count].copy_(pipe.group_sizes[:count], non_blocking=True)
        d2h += count * sizes_host[slot].shape[1] * 8
        done[slot].record()
        return count

    def consume(slot, count):
        done[slot].synchronize()
        return [int(sizes_host[slot][i, L]) for i in range(count)]  # the host reads the results

    def run(t_first, n_steps):
        groups = [(t_first + k, min(G, n_steps - k)) for k in range(0, n_steps, G)]
        pending = None
        for gi, (t0, cnt) in enumerate(groups):
            enqueue(t0, cnt, gi & 1)
            if pending is not None:
                consume(*pending)
            pending = (gi & 1, cnt)
        if pending is not None:
            consume(*pending)

    run(0, W)
    h2d = d2h = 0
    epoch_cache.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(W, K)
    el = time.perf_counter() - t0
    return {"value": K * world / el, "unit": "batches/s",
            "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
            "note": f"per step: pinned H2D of the batch's roots and D2H of its sizes read by the "
                    f"host (launch groups of {G} batches, one group in flight: the host enqueues "
                    f"group k+1 before it waits for group k's sizes), sample+relabel+gather+"
                    f"aggregate on the GPU; the epoch's Knob-1 order is computed on the GPU and "
                    f"read back once per epoch inside the region (wall clock, rank-local x world)"}


def knob_points(bundle, graph, cfg, args, K, flush=False):
    """The paper's knob effect on this workload: batches/s, unique input rows
    and the fused kernel's achieved GB/s at a few (Knob-1, Knob-2) points."""
    import torch
    import paper_2504_18082_b200 as cmb
    pts = []
    L = len(cfg.fanouts)
    # the paper's per-epoch comparisons at p = 0.5 (NORAND 1.69x, MIX-0 1.32x,
    # MIX-50 1.09x over RAND, A100 + model compute) and its best total-training point
    # (MIX-12.5 & p = 1), plus the p = 1 extremes
    paper = {("norand", 0.0, 0.5): 1.69, ("comm", 0.0, 0.5): 1.32, ("comm", 0.5, 0.5): 1.09}
    for mode, mix, p in (("rand", 0.0, 0.5), ("comm", 0.5, 0.5), ("comm", 0.0, 0.5),
                         ("norand", 0.0, 0.5), ("comm", 0.125, 1.0), ("comm", 0.0, 1.0),
                         ("norand", 0.0, 1.0)):
        G = max(1, min(args.batches_per_launch, cmb.MAX_BATCHES_PER_LAUNCH))
        pipe = cmb.BatchedPipeline(graph, torch.from_numpy(bundle.train), cfg.batch_size,
                                   cfg.fanouts, mode=mode, mix=mix, p=p, seed=args.seed, nb=G)
        n = min(K, pipe.n_batches)
        pipe.step_group(range(G))
        s = torch.cuda.current_stream()
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sizes = torch.zeros(n, 2 * L + 1, dtype=torch.int64, device=graph.device)
        evs = []
        scrub = torch.empty(256 << 20, dtype=torch.uint8, device=graph.device) if flush else None
        pool = [pipe.make_events(min(G, n - k0)) for k0 in range(0, n, G)]
        torch.cuda.synchronize()
        e_start.record(s)
        pipe.start_epoch(0)
        for k0 in range(0, n, G):
            el = pool[k0 // G]
            cnt = min(G, n - k0)
            if flush:
                scrub.fill_(k0 & 0xFF)
            ss = pipe.step_group(range(k0, k0 + cnt), events=el)
            evs.append({"sample": (el[0], el[1]),
                        "gather": [(el[2 + 2 * i], el[3 + 2 * i]) for i in range(cnt)]})
            for i, smp in enumerate(ss):
                sizes[k0 + i].copy_(smp.sizes, non_blocking=True)
        e_end.record(s)
        torch.cuda.synchronize()
        ms = e_start.elapsed_time(e_end)
        if flush:
            ms = sum(ev["sample"][0].elapsed_time(ev["gather"][-1][1]) for ev in evs)
        agg = [g0.elapsed_time(g1) for ev in evs for (g0, g1) in ev["gather"]]
        sz = sizes.cpu().numpy()
        alg = [algorithmic_bytes(sz[k, : L + 1], sz[k, L + 1:], cfg.feat_dim, L) for k in range(n)]
        bps = n / (ms * 1e-3)
        pts.append({"knob1": mode + (f"(k={mix})" if mode == "comm" else ""), "p_intra": p,
                    "batches_per_s": bps,
                    "ms_per_epoch": pipe.n_batches / bps * 1e3,
                    "per_epoch_speedup_vs_rand": bps / pts[0]["batches_per_s"] if pts else 1.0,
                    "paper_per_epoch_speedup_context": paper.get((mode, mix, p)),
                    "unique_input_rows": float(sz[:, L].mean()),
                    "gather_aggregate_ms": float(np.mean(agg)),
                    "gather_aggregate_alg_gbps": float(np.mean(alg) / (np.mean(agg) * 1e-3) / 1e9)})
    return pts


def knob_pearson(pts, cfg):
    """The paper's correlation (§6.3): Pearson r between the per-epoch time and
    the per-epoch input-feature volume (unique input rows x 4F bytes x batches) across the knob
    points."""
    t = np.array([q["ms_per_epoch"] for q in pts], dtype=np.float64)
    x = np.array([q["unique_input_rows"] * 4 * cfg.feat_dim for q in pts], dtype=np.float64)
    if t.shape[0] < 3 or np.std(t) == 0 or np.std(x) == 0:
        return None
    return {"r": float(np.corrcoef(t, x)[0, 1]), "points": int(t.shape[0]),
            "x": "unique input-feature bytes per batch", "y": "ms per epoch (a1-a5)"}


def layer_point(bundle, graph, cfg, args, n_batches=64, fo=256):
    """NEXT-4 (R26): the fused a4 + a5 + first GraphSAGE layer kernel
    (cmb_sage_layer_forward, tcgen05 bf16 GEMM, hidden dim 256, bf16 output) timed with
    CUDA events on its stream per batch, next to the a4 + a5 kernel on the same batches.
    Algorithmic bytes per launch: every unique input row once (n_L * 4F), the index streams
    (indptr, last-hop src ids, dst ids) and Y (n_{L-1} * 2 Fo); flops 2 * n_{L-1} * 2F * Fo."""
    import torch
    import paper_2504_18082_b200 as cmb
    L = len(cfg.fanouts)
    F = cfg.feat_dim
    wide = F > 128   # the fused layer keeps K = 2F <= 256 resident; wider rows: cmb_sage_dense_*
    gen = torch.Generator().manual_seed(1)
    ws = torch.randn(F, fo, generator=gen) / np.sqrt(F)
    wn = torch.randn(F, fo, generator=gen) / np.sqrt(F)
    if wide:
        layer = cmb.DenseSageLayer(ws, wn, torch.zeros(fo), relu=True, out_bf16=True,
                                   device=graph.device)
    else:
        layer = cmb.SageLayer(ws, wn, torch.zeros(fo), relu=True, out_bf16=True,
                              device=graph.device)
    # the rest of the paper's 3-layer GraphSAGE: hidden 256 -> 256, last layer 256 -> 48
    # (ogbn-products' 47 classes rounded up to 16), run on hops L-2 .. 0 (reading R29)
    hidden = []
    for l in range(1, len(cfg.fanouts)):
        fout = 48 if l == len(cfg.fanouts) - 1 else fo
        hidden.append(cmb.SageLayer(torch.randn(fo, fout, generator=gen) / np.sqrt(fo),
                                    torch.randn(fo, fout, generator=gen) / np.sqrt(fo),
                                    torch.zeros(fout), relu=fout == fo, out_bf16=fout == fo,
                                    device=graph.device, hidden=True))
    p = cfg.p_intra if args.p is None else args.p
    pipe = cmb.MiniBatchPipeline(graph, torch.from_numpy(bundle.train), cfg.batch_size,
                                 cfg.fanouts, mode=args.mode, mix=args.mix, p=p, seed=args.seed)
    pipe.start_epoch(0)
    smp = pipe.sampler
    out = layer.alloc_out(smp.n_cap[L - 1])
    s = torch.cuda.current_stream()
    n = min(n_batches, pipe.n_batches)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(n)]

    def rest_of_model():
        y = out
        for l, hl in enumerate(hidden):
            y = smp.sage_hidden(hl, L - 2 - l, y)
        return y
    gen_dy = torch.Generator(device=graph.device).manual_seed(2)
    dy = (torch.randn(smp.n_cap[L - 1], fo, generator=gen_dy, device=graph.device) * 0.01
          ).to(torch.bfloat16)
    sizes = torch.zeros(n, 2 * L + 1, dtype=torch.int64, device=graph.device)
    def fwd():
        return smp.sage_dense_layer(layer, out) if wide else smp.sage_layer(layer, out)

    def bwd():   # weight gradients of the same batch
        return (smp.sage_dense_backward(layer, dy, out) if wide else
                smp.sage_layer_backward(layer, dy, out))

    for warm in range(3):
        smp.sample(pipe.batch_roots(warm), p, args.seed, warm)
        fwd()
        bwd()
        rest_of_model()
        smp.gather_aggregate()
    torch.cuda.synchronize()
    for k in range(n):
        smp.sample(pipe.batch_roots(k), p, args.seed, k)
        ev[k][0].record(s)
        fwd()
        ev[k][1].record(s)
        rest_of_model()
        ev[k][4].record(s)
        smp.gather_aggregate()
        ev[k][2].record(s)
        bwd()
        ev[k][3].record(s)
        sizes[k].copy_(smp.sizes, non_blocking=True)
    torch.cuda.synchronize()
    assert smp.status() == 0
    t_layer = np.array([e[0].elapsed_time(e[1]) for e in ev])
    t_agg = np.array([e[4].elapsed_time(e[2]) for e in ev])
    t_rest = np.array([e[1].elapsed_time(e[4]) for e in ev])
    t_bwd = np.array([e[2].elapsed_time(e[3]) for e in ev])
    # R30: the aggregation's backward on layer 2's block (hop L-2) at the hidden width: dX of the
    # layer-1 outputs (n_{L-1} x 256 fp32) += M^T dH (n_{L-2} x 256), for the last batch sampled
    hb = max(0, L - 2)
    szl = sizes[-1].cpu().numpy()
    ndh, nsh = int(szl[hb]), int(szl[hb + 1])
    dH = torch.randn(max(1, smp.n_cap[hb]), fo, device=graph.device)
    dX = torch.zeros(max(1, smp.n_cap[hb + 1]), fo, device=graph.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cmb.sage_mean_backward(smp.indptr[hb], smp.indices[hb], smp.sizes[hb:hb + 1], dH, dX)
    reps = 20
    e0.record(s)
    for _ in range(reps):
        cmb.sage_mean_backward(smp.indptr[hb], smp.indices[hb], smp.sizes[hb:hb + 1], dH, dX)
    e1.record(s)
    torch.cuda.synchronize()
    t_mb = e0.elapsed_time(e1) / reps
    eh = int(szl[L + 1 + hb])
    alg_mb = ndh * fo * 4 + 4 * (ndh + 1) + 4 * eh + 2 * nsh * fo * 4
    sz = sizes.cpu().numpy()
    nL, nd, ed = sz[:, L], sz[:, L - 1], sz[:, L + 1 + L - 1]
    alg = nL * 4 * F + 4 * (nd + 1) + 4 * ed + 4 * nd + nd * 2 * fo
    flops = 2.0 * nd * 2 * F * fo
    peak, peak_src = measured_peak_hbm()
    gbps = float(np.mean(alg) / (np.mean(t_layer) * 1e-3) / 1e9)
    # backward: the same unique rows + index streams, dY and Y read (bf16), partials written and
    # re-read (148 x 2 kh 64 x Fo fp32), dW / db written; flops 2 * n_{L-1} * 2F * Fo
    kh = (F + 63) // 64
    part = 148 * (2 * kh * 64 + 1) * fo * 4
    alg_b = nL * 4 * F + 4 * (nd + 1) + 4 * ed + 4 * nd + 2 * nd * 2 * fo + 2 * part + 4 * (2 * F + 1) * fo
    gbps_b = float(np.mean(alg_b) / (np.mean(t_bwd) * 1e-3) / 1e9)
    if wide:  # unfused: the a4 + a5 bytes (X_in + H written, then read back as the GEMM operand)
        alg = alg + nL * 4 * F + nd * 4 * F + 2 * nd * 2 * 4 * F
    return {"kernel": ("a4+a5 fused gather + cmb_sage_dense_forward (bf16 pack, cuBLASLt bf16 "
                       "GEMM, epilogue): F > 128" if wide else
                       "k_sage_layer (a4+a5+SAGEConv layer 1, tcgen05 bf16, "
                       "cmb_sage_layer_forward)"),
            "out_dim": fo, "out_dtype": "bf16", "relu": True, "batches": int(n),
            "layer_ms": float(np.mean(t_layer)), "gather_aggregate_ms_same_batches": float(np.mean(t_agg)),
            "layers_2_to_L_ms": float(np.mean(t_rest)),
            "model_forward_ms": float(np.mean(t_layer) + np.mean(t_rest)),
            "dst_rows_per_batch": float(nd.mean()), "unique_input_rows_per_batch": float(nL.mean()),
            "algorithmic_bytes_per_launch": float(np.mean(alg)),
            "roofline": {"bound": "hbm", "achieved": gbps, "peak": peak, "peak_source": peak_src,
                         "unit": "GB/s", "frac": gbps / peak},
            "tensor_tflops": float(np.mean(flops) / (np.mean(t_layer) * 1e-3) / 1e12),
            "mean_backward_hidden": {
                "kernel": "k_sage_mean_bwd (cmb_sage_mean_backward, R30), hop L-2 at width 256",
                "dst_rows": ndh, "src_rows": nsh, "edges": eh, "ms": float(t_mb),
                "algorithmic_bytes": float(alg_mb),
                "roofline": {"bound": "hbm", "achieved": float(alg_mb / (t_mb * 1e-3) / 1e9),
                             "peak": peak, "unit": "GB/s",
                             "frac": float(alg_mb / (t_mb * 1e-3) / 1e9 / peak)}},
            "backward": {"kernels": ("cmb_sage_dense_backward (bf16 pack, mask, cuBLASLt bf16 GEMM "
                                     "A^T dZ, fixed-order db)" if wide else
                                     "k_sage_layer_bwd + k_sage_bwd_reduce (cmb_sage_layer_backward)"),
                         "ms": float(np.mean(t_bwd)),
                         "algorithmic_bytes_per_call": float(np.mean(alg_b)),
                         "roofline": {"bound": "hbm", "achieved": gbps_b, "peak": peak,
                                      "unit": "GB/s", "frac": gbps_b / peak},
                         "tensor_tflops": float(np.mean(flops) / (np.mean(t_bwd) * 1e-3) / 1e12)}}


def train_point(bundle, graph, cfg, args, n_batches=48):
    """NEXT-4 (R26-R34): one training step of the paper's 3-layer GraphSAGE (hidden
    256, Adam lr 1e-3, weight decay 5e-4) per mini-batch -- sample (a2 + a3), forward (layer 1
    fused with a4 + a5, hidden layers), softmax cross-entropy, every gradient, Adam, repack --
    timed with CUDA events per batch at the paper's per-epoch comparison points (p = 0.5:
    RAND, COMM-RAND-MIX-50 %, MIX-0 %, NORAND; P:822-825 report 1.09x / 1.32x / 1.69x per-epoch
    TRAINING speedups on A100, averaged over 4 datasets -- context, not a target)."""
    import torch
    import paper_2504_18082_b200 as cmb
    from gen import make_labels, num_classes
    C = num_classes(cfg)
    labels = torch.from_numpy(make_labels(bundle, C)).to(graph.device)
    s = torch.cuda.current_stream()
    points = []
    paper = {("rand", 0.0): None, ("comm", 0.5): 1.09, ("comm", 0.0): 1.32, ("norand", 0.0): 1.69}
    for (mode, mix), ctx in paper.items():
        pipe = cmb.MiniBatchPipeline(graph, torch.from_numpy(bundle.train), cfg.batch_size,
                                     cfg.fanouts, mode=mode, mix=mix, p=0.5, seed=args.seed)
        pipe.start_epoch(0)
        # 4 batches per sampler launch (cmb_sample_blocks_multi), then one training step each
        nbl = 4
        smps = [pipe.sampler] + [cmb.Sampler(graph, cfg.batch_size, cfg.fanouts)
                                 for _ in range(nbl - 1)]
        model = cmb.GraphSAGE(cfg.feat_dim, C, num_layers=len(cfg.fanouts), seed=1,
                              device=graph.device)
        n = (min(n_batches, pipe.n_batches) // nbl) * nbl

        def group(k0):
            cmb.sample_multi(smps, [pipe.batch_roots(k0 + i) for i in range(nbl)],
                             [k0 + i for i in range(nbl)], 0.5, args.seed)

        for w in range(0, 2 * nbl, nbl):  # the first step per sampler captures its CUDA graph
            group(w)
            for sm in smps:
                model.train_step(sm, labels, graph=args.train_graph == "on")
        torch.cuda.synchronize()
        ng = n // nbl
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2 + nbl)] for _ in range(ng)]
        losses = torch.zeros(n, dtype=torch.float64, device=graph.device)
        for q in range(ng):
            ev[q][0].record(s)
            group(q * nbl)
            ev[q][1].record(s)
            for i, sm in enumerate(smps):
                losses[q * nbl + i:q * nbl + i + 1].copy_(
                    model.train_step(sm, labels, graph=args.train_graph == "on"))
                ev[q][2 + i].record(s)
        torch.cuda.synchronize()
        assert all(sm.status() == 0 for sm in smps) and int(model.status.item()) == 0
        t_s = np.array([e[0].elapsed_time(e[1]) for e in ev]) / nbl
        t_t = np.array([e[1].elapsed_time(e[-1]) for e in ev]) / nbl
        per = float(np.mean(t_s + t_t))
        points.append({"knob1": mode + (f"(k={mix})" if mode == "comm" else ""), "p_intra": 0.5,
                       "train_batches_per_s": 1e3 / per, "sample_ms": float(np.mean(t_s)),
                       "train_step_ms": float(np.mean(t_t)),
                       "ms_per_epoch": per * pipe.n_batches, "batches_per_epoch": pipe.n_batches,
                       "loss_first_last": [float(losses[0]), float(losses[-1])],
                       "paper_per_epoch_training_speedup_context": ctx})
    base = points[0]["ms_per_epoch"]
    for pt in points:
        pt["per_epoch_speedup_vs_rand"] = base / pt["ms_per_epoch"]
    return {"model": f"GraphSAGE {len(cfg.fanouts)} layers, hidden 256, {C} classes, Adam",
            "timed": f"{n_batches} consecutive batches of epoch 0 per point, 4 per sampler launch "
                     f"then a training step each (events around the sampler launch and the 4 "
                     f"steps; host enqueue included)",
            "cuda_graph": args.train_graph == "on", "points": points}


def main():
    args = parse()
    if args.impl == "reference" and int(os.environ.get("RANK", "0")) != 0:
        return 0  # the reference arm runs on rank 0 only; the other ranks exit without work
    if args.impl == "cmb" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    from gen import CONFIGS, generate
    cfg = CONFIGS[args.config]
    if args.impl == "cmb" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # ranks start together; rank 0 generates (or loads) the bundle first, the others then
        # read the generator's on-disk cache instead of generating it concurrently
        import torch.distributed as dist
        world, rank = init_ranks()[:2]
        if rank == 0:
            generate(cfg, features=False)
        dist.barrier()
    bundle = generate(cfg)
    if args.impl == "reference":
        return run_reference(args, bundle)
    if args.shard != "none":
        return run_sharded(args, bundle)
    return run_cmb(args, bundle)


if __name__ == "__main__":
    sys.exit(main())
