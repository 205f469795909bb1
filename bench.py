#!/usr/bin/env python
"""bench.py -- APS gradient-sync throughput on B200 (BASELINE.json metric
"APS sync GB/s (fp32-equiv) & % NVLink/HBM roofline at 1/2/4/8 B200").

One step = one whole APS synchronisation of the
config-2 workload: ResNet-50 gradient shapes (161 tensors, 25,557,032 fp32
elements per rank), format 1/5/2, synthetic seeded gradients (synthetic/),
resident in HBM before the timed region.  At N = 1 the step is the fused
single launch (abs-max -> f~ -> Cast -> pack -> Cast back -> unscale); at N > 1
(one process per GPU) it adds the exponent MAX exchange and the packed
reduce-scatter / all-gather (peer-memory transport by default, or the NCCL
send/recv ring).

Timing (the headline): K syncs back to back between ONE pair of CUDA events on
the library's stream, rotating over S >= 3 buffer sets (each: gradients,
outputs, packed codes; S x 230 MB > the 126 MB L2), so every step's deferred
write-backs land inside the timed region -- steady state.  Max over ranks.
  value        = N x 4 L / t_sync   (whole-job fp32-equivalent GB/s: N ranks' gradients)
  per_rank     = 4 L / t_sync       (SURVEY 8(d)'s metric; BASELINE.md's ideal 0.8-0.9 TB/s at p = 8)
Beside it: the L2-flushed single-step time, a per-phase breakdown through the four
separate calls, the roofline of the dominant kernel, e2e through aps_sync_host
(pinned host buffers, copies inside), the CPU oracle (all host cores), and at
N > 1 the bit-exact parity check of the synced data against the oracle (both
transports) and the NCCL / p2p reference points.

`python bench.py --gpus N` without torchrun re-launches itself under
`torch.distributed.run` with N processes.  `--impl reference` times the CPU
oracle (the reference arm of this paper-only tier).  `--config c5` runs the
message-size sweep, `--formats a,b:c,d` the format sweep (C4).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "APS sync GB/s (fp32-equiv) & % NVLink/HBM roofline at 1/2/4/8 B200"
UNIT = "GB/s"
NVLINK_MEASURED = 770.0   # B200_PROFILING.md: measured peer copy per direction (nominal 900)
NVLINK_NOMINAL = 900.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="aps", choices=["aps", "reference"])
    ap.add_argument("--format", default="5,2")
    ap.add_argument("--formats", default=None,
                    help="C4 format sweep, e.g. 3,0:5,2:4,3:5,6:5,10 (adds 'format_sweep' to the line)")
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "res5c", "c5"])
    ap.add_argument("--sets", type=int, default=3, help="rotating buffer sets of the steady-state timing")
    ap.add_argument("--no-hw", action="store_true", help="generic bit-arithmetic codec instead of cvt")
    ap.add_argument("--hybrid", action="store_true",
                    help="hybrid precision (P:545): last layer (final two tensors) in FP32 (8,23), the rest --format")
    ap.add_argument("--hybrid-last", default="8,23", help="format of the last layer under --hybrid")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--phase-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "peer"],
                    help="N > 1: NCCL send/recv ring, or the peer-memory (CUDA IPC / NVLink) owner-computes "
                         "kernel; auto = peer, falling back to the NCCL ring if the IPC mapping fails")
    ap.add_argument("--group-k", type=int, default=1,
                    help="hierarchical all-reduce group size (P:509-541; needs --transport peer when != 1, N)")
    ap.add_argument("--acc", default=None, help="accumulator format e,m (CPD, P:660-678; needs --transport peer)")
    ap.add_argument("--kahan", action="store_true", help="Kahan-compensated accumulation (needs --transport peer)")
    ap.add_argument("--no-peer-sim", action="store_true", help="skip the simulated p = 8 peer all-reduce phase")
    ap.add_argument("--graph", type=int, default=None,
                    help="1: time replays of each buffer set's sync captured in a CUDA graph; default: on for "
                         "N > 1 (a sync is ~8 launches), off for N = 1 (one launch)")
    return ap.parse_args()


# ---------------------------------------------------------------------------- plumbing
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args) -> int:
    """--gpus N without torchrun: re-run this script under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def workload(cfg):
    import synthetic
    if cfg == "c2":
        return "resnet50_grads", synthetic.RESNET50_NUMELS
    if cfg == "c3":
        return "bert_large_grads", synthetic.BERT_LARGE_NUMELS
    return "resnet50_res5c_merged", synthetic.RES5C_NUMELS


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of each kernel role from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")  # written by scripts/ncu_summary.py
    try:
        return json.load(open(p))
    except Exception:
        return {}


def ncu_traffic_steady():
    """DRAM bytes per fused launch in steady state (ncu application replay, caches as the
    program leaves them): profiles/ncu_traffic_steady.json."""
    try:
        return int(json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic_steady.json")))
                   ["dram_bytes_per_launch_median"])
    except Exception:
        return None


def host_cpu():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return os.cpu_count() or 1, model


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks and throttle reasons
    during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------- CPU oracle legs
def oracle_sample(numels, p, budget_s, n_threads):
    """A prefix of the layer list whose oracle sync (p simulated ranks, n_threads)
    takes about budget_s; returns (prefix numels, per-element seconds)."""
    import oracle
    import synthetic
    oracle.build()
    probe = numels[:8]
    g = synthetic.make_grads(probe, p)
    t0 = time.perf_counter()
    oracle.aps_sync(g, 5, 2, want_packed=False, n_threads=n_threads)
    per_elem = (time.perf_counter() - t0) / (p * sum(probe))
    sample, tot = [], 0
    for n in numels:
        if sample and (tot + n) * p * per_elem > budget_s:
            break
        sample.append(n)
        tot += n
    return sample, per_elem


def cpu_oracle_run(numels, e, m, p, budget_s=20.0, min_s=10.0):
    """The CPU oracle (plain C) on all host cores, on a bounded sample of the
    workload, p simulated ranks: a prefix of the layer list sized to ~budget_s of
    work, and -- when the whole workload takes less -- whole syncs repeated until
    at least min_s of CPU work (the 10-30 s the contract asks for)."""
    import oracle
    import synthetic
    cores, model = host_cpu()
    sample, _ = oracle_sample(numels, p, budget_s, cores)
    grads = synthetic.make_grads(sample, p)
    t0 = time.perf_counter()
    r = oracle.aps_sync(grads, e, m, want_packed=False, n_threads=cores)
    t1 = time.perf_counter() - t0
    assert r.rc == 0
    reps = 1 + max(0, int((min_s - t1) / max(t1, 1e-3)))
    t = t1
    if reps > 1:
        t0 = time.perf_counter()
        for _ in range(reps - 1):
            oracle.aps_sync(grads, e, m, want_packed=False, n_threads=cores)
        t += time.perf_counter() - t0
    L = sum(sample)
    desc = (f"first {len(sample)} of {len(numels)} layers ({L} of {sum(numels)} elements) x {p} simulated "
            f"rank(s), full oracle aps_sync (FindMaxExp, MAX, cast, ring, unscale), {reps} sync(s), {cores} threads")
    # single-threaded beside it: a prefix of ~6 s of work
    s1, _ = oracle_sample(numels, p, 6.0, 1)
    g1 = synthetic.make_grads(s1, p)
    t0 = time.perf_counter()
    oracle.aps_sync(g1, e, m, want_packed=False, n_threads=1)
    t1s = time.perf_counter() - t0
    single = {"value": round(4 * sum(s1) / t1s / 1e9, 6), "unit": UNIT, "cores": 1, "seconds": round(t1s, 3),
              "sample": f"first {len(s1)} layers ({sum(s1)} elements) x {p} simulated rank(s), 1 thread"}
    return {"value": round(4 * L * reps / t / 1e9, 6), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
            "seconds": round(t, 3), "syncs": reps, "cpu_model": model, "nproc": cores,
            "single_thread": single,
            "note": "per-rank fp32-equivalent GB/s (4 L / t, as the GPU line's per_rank)"}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    e, m = map(int, args.format.split(","))
    name, numels = workload(args.config if args.config != "c5" else "c2")
    p = max(args.gpus, world)
    import oracle
    import synthetic
    cores, model = host_cpu()
    per_step_budget = max(1.0, min(30.0, 150.0 / (args.steps + args.warmup)))
    sample, _ = oracle_sample(numels, p, per_step_budget, cores)
    grads = synthetic.make_grads(sample, p)
    for _ in range(args.warmup):
        oracle.aps_sync(grads, e, m, want_packed=False, n_threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.aps_sync(grads, e, m, want_packed=False, n_threads=cores)
        times.append(time.perf_counter() - t0)
    L = sum(sample)
    tot_t = sum(times)
    value = p * 4 * L * args.steps / tot_t / 1e9   # whole job: p ranks' gradients, as the GPU arm's value
    sample_desc = (f"first {len(sample)} of {len(numels)} layers ({L} elements) x {p} simulated ranks per step, "
                   f"{cores} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (oracle)",
        "data": "synthetic", "config": {"workload": name, "format": f"1/{e}/{m}", "ranks": p,
                                        "sample": sample_desc},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample_desc, "cpu_model": model},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------- the GPU arm
class Bench:
    def __init__(self, args):
        import torch
        import paper_1911_08907_b200 as aps
        self.torch, self.aps, self.args = torch, aps, args
        self.world, self.rank, local = dist_env()
        # APS_BENCH_SAME_GPU=1 (plumbing check only, no valid numbers): every rank on cuda:0,
        # a gloo group, no NCCL communicator, the peer transport across processes
        self.same_gpu = os.environ.get("APS_BENCH_SAME_GPU") == "1" and self.world > 1
        if self.same_gpu:
            local = 0
            args.transport = "peer"
        self.local = local
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.comm = None
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            self.dist = dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if self.same_gpu:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
                uid = [aps.nccl_unique_id() if self.rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                self.comm = aps.nccl_comm_init(uid[0], self.world, self.rank)
        self.stream = torch.cuda.Stream(self.dev)   # a non-default stream (CUDA-graph capture needs one)
        torch.cuda.set_stream(self.stream)
        os.environ.setdefault("APS_PEER_TIMEOUT_S", "20")  # a failed peer wait must not stall the bench

    # -------------------------------------------------------------- helpers
    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cpu" if self.same_gpu else self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def all_ok(self, ok: bool) -> bool:
        if not self.dist:
            return ok
        t = self.torch.tensor([1.0 if ok else 0.0], dtype=self.torch.float64,
                              device="cpu" if self.same_gpu else self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return t.item() == 1.0

    def make_ctx(self, e, m, numels, fmts, transport, stream=None):
        aps, a = self.aps, self.args
        ctx = aps.ApsContext(e, m, numels, world_size=self.world, rank=self.rank,
                             nccl_comm=self.comm if transport == "nccl" else None,
                             stream=stream or self.stream, device=self.dev, hw_convert=not a.no_hw, formats=fmts)
        if self.world > 1:
            if transport == "peer":
                ctx.connect_peers()
            ctx.set_reduction(a.group_k, tuple(map(int, a.acc.split(","))) if a.acc else None, a.kahan)
        return ctx

    def pick_transport(self, e, m, numels, fmts):
        """auto: the peer transport if every rank can map every workspace, else the NCCL ring."""
        t = self.args.transport
        if self.world == 1:
            return "none"
        if t in ("auto", "peer"):
            try:
                c = self.make_ctx(e, m, numels[:1], None, "peer")
                c.close()
                return "peer"
            except Exception as exc:
                if t == "peer" or self.comm is None:
                    raise
                print(f"[bench] peer transport unavailable ({exc}); using the NCCL ring", file=sys.stderr)
        return "nccl"

    # -------------------------------------------------------------- parity vs the oracle
    def parity(self, e, m, numels, fmts, transport, sets):
        """One sync of the bench data through `transport`, checked bit-exactly against the
        CPU oracle run over all `world` ranks' synthetic gradients on rank 0: f~, the
        reduced packed codes (every rank's equal to rank 0's) and every output of rank 0."""
        import numpy as np
        torch = self.torch
        g, o = sets[0][0], sets[0][1]
        ctx = self.make_ctx(e, m, numels, fmts, transport)
        ctx.sync_out(g, o, average=True)
        st = ctx.status_sync()
        packed = ctx.packed().cpu().numpy()
        digest = int(np.frombuffer(packed.tobytes(), dtype=np.uint8).astype(np.uint64).dot(
            np.arange(1, packed.size + 1, dtype=np.uint64) % 65521))
        ft = ctx.scales()
        outs = [x.cpu().numpy() for x in o]
        self.barrier()
        ctx.close()
        # every rank's reduced codes must be identical (O9): compare digests
        digests = [digest]
        if self.dist:
            digests = [None] * self.world
            self.dist.all_gather_object(digests, (digest, st))
            sts = [d[1] for d in digests]
            digests = [d[0] for d in digests]
        else:
            sts = [st]
        res = {"transport": transport, "ok": False}
        if self.rank == 0:
            import oracle
            import synthetic
            cores, _ = host_cpu()
            grads = synthetic.make_grads(numels, self.world)
            t0 = time.perf_counter()
            if fmts:
                ref = oracle.aps_sync_mixed(grads, fmts, average=1)
            elif self.args.group_k != 1 or self.args.acc or self.args.kahan:
                acc = tuple(map(int, self.args.acc.split(","))) if self.args.acc else None
                ref = oracle.aps_sync_ex(grads, e, m, average=1, group_k=self.args.group_k, acc=acc,
                                         kahan=int(self.args.kahan))
            else:
                ref = oracle.aps_sync(grads, e, m, average=1, want_packed=False, n_threads=cores)
            t_or = time.perf_counter() - t0
            ok_ft = bool(np.array_equal(ft, ref.ftilde))
            ok_codes = bool(np.array_equal(packed, ref.reduced))
            ok_same = len(set(digests)) == 1
            bad_out = sum(int((a.view(np.uint32) != b.view(np.uint32)).sum()) for a, b in zip(outs, ref.out))
            res.update({"ok": ok_ft and ok_codes and ok_same and bad_out == 0 and all(s == 0 for s in sts),
                        "ftilde": ok_ft, "reduced_codes": ok_codes, "ranks_identical": ok_same,
                        "outputs_mismatched": bad_out, "elements_checked": int(sum(numels)),
                        "status": sts, "oracle_s": round(t_or, 2), "ranks": self.world})
        ok = self.all_ok(res["ok"] if self.rank == 0 else True)
        res["ok"] = ok
        return res

    # -------------------------------------------------------------- N > 1 reference points
    def nccl_refs(self, L, packed_bytes, iters=20):
        """fp32 / fp16 ncclAllReduce on the same L (the paper's baseline is the fp16 all-reduce,
        P:636-640; its cost model 8L vs 16L bits) and a large ring send/recv (the
        practical per-direction link ceiling)."""
        torch, dist = self.torch, self.dist
        out = {}
        p = self.world

        def time_op(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            self.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            for _ in range(iters):
                fn()
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            return self.max_over_ranks(e0.elapsed_time(e1) / iters)

        for name, dt, nb in (("nccl_allreduce_fp32", torch.float32, 4), ("nccl_allreduce_fp16", torch.float16, 2)):
            x = torch.ones(L, dtype=dt, device=self.dev)
            ms = time_op(lambda: dist.all_reduce(x))
            out[name] = {"us": round(ms * 1e3, 1), "per_rank_GBps_fp32eq": round(4 * L / (ms * 1e-3) / 1e9, 1),
                         "busBW_GBps": round(2 * (p - 1) / p * nb * L / (ms * 1e-3) / 1e9, 1)}
            del x
        nbytes = max(packed_bytes, 256 << 20)
        sb = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        rb = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)

        def ring():
            ops = [dist.P2POp(dist.isend, sb, (self.rank + 1) % p), dist.P2POp(dist.irecv, rb, (self.rank - 1) % p)]
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        ms = time_op(ring)
        out["p2p_ring_sendrecv"] = {"bytes": nbytes, "us": round(ms * 1e3, 1),
                                    "GBps_per_direction": round(nbytes / (ms * 1e-3) / 1e9, 1)}
        return out

    # -------------------------------------------------------------- the measurement of one format
    def measure(self, e, m, numels, fmts, transport, want_graph, steps, warmup, sets_n):
        torch, aps, args = self.torch, self.aps, self.args
        import synthetic
        L = sum(numels)
        host = [synthetic.layer_grad(self.rank, l, n) for l, n in enumerate(numels)]
        sets = []
        for _ in range(sets_n):
            g = [torch.from_numpy(a).to(self.dev) for a in host]
            o = [torch.empty_like(x) for x in g]
            sets.append((g, o, aps.ApsContext.ptr_array(g), aps.ApsContext.ptr_array(o)))
        ctxs = [self.make_ctx(e, m, numels, fmts, transport) for _ in range(sets_n)]
        graphs = None
        note = None
        if want_graph:
            try:
                graphs = [c.capture_sync(s[0], s[1], average=True) for c, s in zip(ctxs, sets)]
            except Exception as exc:
                note = f"capture failed ({exc}); plain calls timed"
                graphs = None
                torch.cuda.synchronize()

        def step(k):
            i = k % sets_n
            if graphs:
                graphs[i].replay()
            else:
                ctxs[i].sync_out(sets[i][2], sets[i][3], average=True)

        for k in range(max(warmup, 3) * sets_n):
            step(k)
        torch.cuda.synchronize()
        st = [c.status_sync() for c in ctxs]
        if not self.all_ok(all(s == 0 for s in st)):
            raise SystemExit(f"sync reported status {st} on synthetic data")
        # ---- steady state: K syncs back to back between one event pair
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.barrier()
        torch.cuda.synchronize()
        with ClockSampler(self.local) as clk:
            e0.record(self.stream)
            for k in range(steps):
                step(k)
            e1.record(self.stream)
            torch.cuda.synchronize()
        self.barrier()
        ms = self.max_over_ranks(e0.elapsed_time(e1) / steps)
        # ---- L2-flushed single steps (the round-1 method): each step alone, cold L2
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=self.dev)
        flush_rd = torch.zeros(256 << 20, dtype=torch.uint8, device=self.dev)
        KF = min(steps, 20)
        fev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(KF)]
        for k in range(KF):
            flush.zero_()
            flush_rd.sum(dtype=torch.int32)
            fev[k][0].record(self.stream)
            step(0)
            fev[k][1].record(self.stream)
        torch.cuda.synchronize()
        flushed_ms = self.max_over_ranks(statistics.median(fev[k][0].elapsed_time(fev[k][1]) for k in range(KF)))
        # ---- per-phase breakdown through the four separate calls (flushed; these are the
        # kernels of the N > 1 path)
        c0, (g0, o0, gp, op) = ctxs[0], sets[0]
        KP = args.phase_steps
        pev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(KP)]

        def calls(ev):
            ev[0].record(self.stream)
            c0.layer_scales(gp)
            ev[1].record(self.stream)
            c0.quantize_pack(gp)
            ev[2].record(self.stream)
            c0.allreduce()
            ev[3].record(self.stream)
            c0.unscale(op, average=True)
            ev[4].record(self.stream)
        if graphs:
            c0.set_graph_safe(False)
        for _ in range(3):
            calls(pev[0])
        torch.cuda.synchronize()
        for k in range(KP):
            flush.zero_()
            flush_rd.sum(dtype=torch.int32)
            calls(pev[k])
        torch.cuda.synchronize()
        phase_ms = [statistics.median(pev[k][i].elapsed_time(pev[k][i + 1]) for k in range(KP)) for i in range(4)]
        phase_ms = [self.max_over_ranks(x) for x in phase_ms]
        del flush, flush_rd
        ok = all(c.status_sync() == 0 for c in ctxs)
        for c in ctxs:
            if self.dist:
                self.barrier()
            c.close()
        return {"ms": ms, "flushed_ms": flushed_ms, "phase_ms": phase_ms, "graph": graphs is not None,
                "graph_note": note, "clocks": clk.summary(), "ok": ok, "sets": sets, "host": host}

    # -------------------------------------------------------------- e2e through aps_sync_host
    def e2e(self, e, m, numels, fmts, transport, host):
        torch = self.torch
        L = sum(numels)
        slots = 2   # two contexts on two streams alternate: step k's D2H overlaps step k+1's H2D
        ectx = [self.make_ctx(e, m, numels, fmts, transport, stream=self.stream if s == 0 else torch.cuda.Stream(self.dev))
                for s in range(slots)]
        # flat pinned host buffers with per-layer views (every ResNet-50 / BERT layer size is a
        # multiple of 4 elements: 16-byte aligned views), as a training loop's flat gradient
        # buffer; aps_sync_host then moves each direction in one copy
        offs = [0]
        for n in numels:
            offs.append(offs[-1] + (n + 3) // 4 * 4)

        def views(flat):
            return [flat[offs[l]:offs[l] + n] for l, n in enumerate(numels)]
        hin, hout, dgr = [], [], []
        for _ in range(slots):
            fi = torch.empty(offs[-1], dtype=torch.float32).pin_memory()
            for v, a in zip(views(fi), host):
                v.copy_(torch.from_numpy(a))
            hin.append(views(fi))
            hout.append(views(torch.empty(offs[-1], dtype=torch.float32).pin_memory()))
            dgr.append(views(torch.empty(offs[-1], dtype=torch.float32, device=self.dev)))
        for sl in range(slots):
            for _ in range(2):
                ectx[sl].sync_host(hin[sl], dgr[sl], hout[sl], average=True)
        torch.cuda.synchronize()
        E = max(self.args.e2e_steps, slots)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.barrier()
        e0.record(self.stream)
        for c2 in ectx[1:]:
            c2.stream.wait_event(e0)
        for k in range(E):
            sl = k % slots
            ectx[sl].sync_host(hin[sl], dgr[sl], hout[sl], average=True)
        for c2 in ectx[1:]:
            ev = torch.cuda.Event()
            ev.record(c2.stream)
            self.stream.wait_event(ev)
        e1.record(self.stream)
        torch.cuda.synchronize()
        ms = self.max_over_ranks(e0.elapsed_time(e1) / E)
        for c2 in ectx:
            self.barrier()
            c2.close()
        return {"value": round(self.world * 4 * L / (ms * 1e-3) / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": 4 * L, "d2h_bytes_per_step": 4 * L, "ms_per_step": round(ms, 4),
                "api": "aps_sync_host", "pipelined_contexts": slots}

    # -------------------------------------------------------------- simulated p = 8 peer reduce (N = 1)
    def peer_sim(self, e, m, numels):
        torch, aps = self.torch, self.aps
        import synthetic
        P8 = 8
        ss = torch.cuda.Stream(self.dev)
        sim = [aps.ApsContext(e, m, numels, world_size=P8, rank=r, stream=ss, device=self.dev,
                              hw_convert=not self.args.no_hw) for r in range(P8)]
        aps.sim_connect(sim)
        sgr = [[torch.from_numpy(synthetic.layer_grad(r, l, n)).to(self.dev) for l, n in enumerate(numels)]
               for r in range(P8)]
        torch.cuda.synchronize()
        aps.sim_layer_scales(sim, sgr)
        for r in range(P8):
            sim[r].quantize_pack(sgr[r])
        for _ in range(2):
            aps.sim_allreduce(sim)
            for r in range(P8):
                sim[r].quantize_pack(sgr[r])
        torch.cuda.synchronize()
        pg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(pg, stream=ss):
            aps.sim_allreduce(sim)
        pg.replay()
        torch.cuda.synchronize()
        pe = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 20
        with torch.cuda.stream(ss):
            pe[0].record(ss)
            for _ in range(reps):
                pg.replay()
            pe[1].record(ss)
        torch.cuda.synchronize()
        ms = pe[0].elapsed_time(pe[1]) / reps
        _, pb = aps.layout(P8, e, m, numels)
        byts = P8 * 2 * pb
        for c in sim:
            c.close()
        return {"us": round(ms * 1e3, 2), "algorithmic_bytes": int(byts),
                "GB/s": round(byts / (ms * 1e-3) / 1e9, 1), "frac": round(byts / (ms * 1e-3) / 1e9 / peaks()[0], 4),
                "note": "aps_sim_allreduce of 8 simulated ranks through the peer transport on one device "
                        "(CUDA-graph replay): 8 owner-computes reduce kernels (each loads the 8 ranks' codes of "
                        "its chunk, folds in ring order, stores into all 8 buffers) + epoch-flag kernels; every "
                        "byte is local HBM here"}

    # -------------------------------------------------------------- launches per step
    def launches(self, numels, fmts, e, m, transport):
        G = len(set(fmts)) if fmts else 1
        if self.world == 1:   # one fused launch per format group; two formats share one launch
            return 1 if G <= 2 else G
        if transport == "peer":   # absmax, E exchange, G quantise, ready + done flag kernels, own-chunk runs, G unscale
            runs = format_runs(numels, fmts or [(e, m)] * len(numels), self.world, (self.rank + 2) % self.world)[0]
            return 1 + 1 + 2 * G + 2 + runs
        # NCCL ring: absmax + G quantise + one reduce launch per format run per ring step + G unscale
        return 1 + 2 * G + sum(format_runs(numels, fmts or [(e, m)] * len(numels), self.world, self.rank))

    # -------------------------------------------------------------- main
    def run(self):
        args, torch = self.args, self.torch
        e, m = map(int, args.format.split(","))
        b = 1 + e + m
        name, numels = workload(args.config)
        L = sum(numels)
        last = tuple(map(int, args.hybrid_last.split(",")))
        fmts = [(e, m)] * (len(numels) - 2) + [last] * 2 if args.hybrid else None
        code_bytes = sum(n * (1 + f[0] + f[1]) for n, f in zip(numels, fmts)) / 8 if fmts else L * b / 8
        transport = self.pick_transport(e, m, numels, fmts)
        want_graph = args.graph if args.graph is not None else int(self.world > 1)
        r = self.measure(e, m, numels, fmts, transport, want_graph, args.steps, args.warmup, args.sets)
        ms = r["ms"]
        T, packed_bytes = (self.aps.layout_mixed(self.world, numels, fmts) if fmts
                           else self.aps.layout(self.world, e, m, numels))
        # ---- parity of the timed data against the oracle (N > 1: both transports)
        parity = None
        if not args.no_parity:
            parity = {"checked": []}
            tlist = [transport] if self.world == 1 else (["peer", "nccl"] if self.comm is not None else ["peer"])
            for tp in tlist:
                parity["checked"].append(self.parity(e, m, numels, fmts, tp if tp != "none" else "none",
                                                     r["sets"]))
            parity["ok"] = all(x["ok"] for x in parity["checked"])
            parity["transport_timed"] = transport
        # ---- rooflines
        peak, peak_kind = peaks()
        pm = r["phase_ms"]
        kern = {
            "absmax_exp": (pm[0], 4 * L),
            "quant_pack": (pm[1], 4 * L + code_bytes),
            "unpack_unscale": (pm[3], code_bytes + 4 * L),
        }
        if self.world > 1:
            kern["allreduce"] = (pm[2], 2 * (self.world - 1) / self.world * packed_bytes)
        phases = {}
        for k, (pms, byts) in kern.items():
            gbs = byts / (pms * 1e-3) / 1e9
            ref_peak = NVLINK_MEASURED if k == "allreduce" else peak
            phases[k] = {"us": round(pms * 1e3, 2), "algorithmic_bytes": int(byts), "GB/s": round(gbs, 1),
                         "frac": round(gbs / ref_peak, 4)}
        if self.world > 1:
            phases["allreduce"]["note"] = ("busBW = 2(p-1)/p x packed bytes / t; frac of the measured 770 GB/s "
                                           "per direction (nominal 900)")
        traffic = ncu_traffic() if (args.config == "c2" and (e, m) == (5, 2) and not args.no_hw and not fmts) else {}
        traffic_steady = (ncu_traffic_steady() if (args.config == "c2" and (e, m) == (5, 2) and not args.no_hw
                                                   and not fmts) else None)
        if self.world == 1:
            # one fused launch per step; NECESSARY bytes: one fp32 read + codes + fp32 output (the
            # abs-max pass and the quantise pass read the same gradients; the second read is L2)
            dbytes = 8 * L + code_bytes
            achieved = dbytes / (ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "frac_vs_8TBps_spec": round(achieved / 8000.0, 4),
                    "traffic": traffic.get("fused_p1"),
                    "kernel": "fused_cw_kernel (a1 + a3 + a4 + a7, one launch)",
                    "algorithmic_bytes_per_launch": int(dbytes),
                    "algorithmic_bytes_rule": "8 L + code bytes: one fp32 read, the packed codes, one fp32 write",
                    "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                    "timing": "steady state (back-to-back syncs, rotating buffer sets > L2)",
                    "traffic_note": ("traffic: one ncu --set full capture (cold caches: ~55 MB of the launch's "
                                     "writes are still dirty in L2 at kernel end)"),
                    "traffic_steady_state": traffic_steady}
        else:
            dom = max(kern, key=lambda k: kern[k][0])
            dms, dbytes = kern[dom]
            achieved = dbytes / (dms * 1e-3) / 1e9
            if dom == "allreduce":
                roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_MEASURED, "unit": "GB/s",
                        "frac": round(achieved / NVLINK_MEASURED, 4), "traffic": None, "kernel": dom,
                        "peak_kind": "measured NVLink peer copy per direction (B200_PROFILING.md; nominal 900)"}
            else:
                roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                        "frac": round(achieved / peak, 4), "traffic": traffic.get(dom), "kernel": dom,
                        "algorithmic_bytes_per_launch": int(dbytes),
                        "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)"}
        if roof["frac"] > 1.0:
            roof["flag"] = "frac > 1: the algorithmic bytes overstate what the kernel moves, or the peak is low"
        if roof.get("traffic") and roof.get("algorithmic_bytes_per_launch"):
            roof["traffic_vs_algorithmic"] = round(roof["traffic"] / roof["algorithmic_bytes_per_launch"], 3)
        extra = {}
        if self.world == 1 and not args.no_peer_sim and not fmts and args.config != "c3":
            phases["peer_allreduce_p8_sim"] = self.peer_sim(e, m, numels)
        if self.world > 1 and self.comm is not None:
            extra["references"] = self.nccl_refs(L, packed_bytes)
            # the other transport timed too (the NCCL send/recv ring is north_star's design, the
            # peer-memory kernel the default): sync time and the all-reduce phase's busBW of each
            other = "nccl" if transport == "peer" else "peer"
            tr = {transport: {"sync_us": round(ms * 1e3, 2), "allreduce_us": round(r["phase_ms"][2] * 1e3, 2),
                              "busBW_GBps": round(2 * (self.world - 1) / self.world * packed_bytes
                                                  / (r["phase_ms"][2] * 1e-3) / 1e9, 1)}}
            try:
                ro = self.measure(e, m, numels, fmts, other, want_graph, max(20, args.steps // 2), 3, args.sets)
                tr[other] = {"sync_us": round(ro["ms"] * 1e3, 2), "allreduce_us": round(ro["phase_ms"][2] * 1e3, 2),
                             "busBW_GBps": round(2 * (self.world - 1) / self.world * packed_bytes
                                                 / (ro["phase_ms"][2] * 1e-3) / 1e9, 1), "ok": ro["ok"]}
                del ro["sets"], ro["host"]
            except (Exception, SystemExit) as exc:   # reported, never fatal (every rank raises together)
                tr[other] = {"error": str(exc)[:200]}
            extra["transports"] = tr
        e2e = self.e2e(e, m, numels, fmts, transport, r["host"])
        del r["sets"]
        fsweep = None
        if args.formats:
            fsweep = []
            for fs in args.formats.split(":"):
                fe, fm = map(int, fs.split(","))
                rr = self.measure(fe, fm, numels, None, transport, want_graph, max(20, args.steps // 2), 3, args.sets)
                del rr["sets"]
                fb = 1 + fe + fm
                nb = 8 * L + L * fb / 8
                fsweep.append({"format": f"1/{fe}/{fm}", "bits": fb, "sync_us": round(rr["ms"] * 1e3, 2),
                               "per_rank_GBps": round(4 * L / (rr["ms"] * 1e-3) / 1e9, 1),
                               "hbm_frac_necessary_bytes": round(nb / (rr["ms"] * 1e-3) / 1e9 / peak, 4)
                               if self.world == 1 else None,
                               "phases_us": {k: round(x * 1e3, 2) for k, x in
                                             zip(("absmax_exp", "quant_pack", "allreduce", "unpack_unscale"),
                                                 rr["phase_ms"])},
                               "ok": rr["ok"]})
        result = {
            "metric": METRIC, "value": round(self.world * 4 * L / (ms * 1e-3) / 1e9, 3), "unit": UNIT,
            "n_gpus": self.world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32",
            "per_rank": {"value": round(4 * L / (ms * 1e-3) / 1e9, 3), "unit": UNIT, "sync_us": round(ms * 1e3, 2),
                         "note": "SURVEY 8(d)'s metric 4 L / t_sync; value = n_gpus x this (whole job)"},
            "wire_dtype": (f"{b}-bit 1/{e}/{m} codes, last layer 1/{last[0]}/{last[1]}" if fmts else f"{b}-bit 1/{e}/{m} codes"),
            "data": "synthetic (seeded normal per layer, binade spread 2^-24..2^-4, 0.5% zeros)",
            "config": {"workload": name, "format": f"1/{e}/{m}" + (f" + last layer 1/{last[0]}/{last[1]} (hybrid)" if fmts else ""),
                       "n_layers": len(numels), "elements": L, "ranks": self.world,
                       "hw_convert": (not args.no_hw) and (e, m) in ((5, 2), (4, 3), (5, 10), (8, 7), (8, 23)),
                       "l2": (f"inputs larger than L2: {args.sets} rotating buffer sets (gradients + outputs + "
                              f"packed codes, {args.sets * (8 * L + code_bytes) / 1e6:.0f} MB) timed back to back"),
                       "parallelism": f"dp{self.world}", "packed_bytes": packed_bytes,
                       "cuda_graph": r["graph"], "transport": transport},
            "flushed": {"us": round(r["flushed_ms"] * 1e3, 2),
                        "note": "median single sync after a 256 MiB L2 flush (write + read), round-1 method"},
            "roofline": roof, "phases": phases, "gpu_launches": self.launches(numels, fmts, e, m, transport) * args.steps,
            "e2e": e2e, "clocks": r["clocks"],
        }
        if r["graph_note"]:
            result["config"]["cuda_graph_note"] = r["graph_note"]
        if parity is not None:
            result["parity"] = parity
        if self.world > 1:
            result["config"]["ring"] = (
                "peer memory (CUDA IPC over NVLink): owner-computes reduce + fused all-gather, E max over peer memory"
                if transport == "peer" else "ncclSend/ncclRecv reduce-scatter + ncclAllGather, int32 MAX all-reduce")
            result["config"]["reduction"] = {"group_k": args.group_k, "acc": args.acc or f"{e},{m}",
                                             "kahan": bool(args.kahan)}
        if self.same_gpu:
            result["config"]["same_gpu_plumbing"] = "APS_BENCH_SAME_GPU=1: every rank on cuda:0 -- numbers invalid"
        result.update(extra)
        if fsweep is not None:
            result["format_sweep"] = fsweep
        if self.rank == 0:
            if not args.no_cpu_baseline:
                result["cpu_baseline"] = cpu_oracle_run(numels, e, m, self.world, budget_s=20.0 if self.world == 1 else 25.0)
            print(json.dumps(result), flush=True)
        self.close()

    # -------------------------------------------------------------- C5: message-size sweep
    def run_c5(self):
        """One tensor, (5,2), packed 8-bit sizes 1 KB .. 1 GB in x4 steps:
        the APS sync vs fp32 / fp16 ncclAllReduce on the same element count; busBW of the
        packed all-reduce phase and where it crosses 70 % of the link."""
        args, torch, aps = self.args, self.torch, self.aps
        e, m = map(int, args.format.split(","))
        b = 1 + e + m
        transport = self.pick_transport(e, m, [1024], None)
        want_graph = args.graph if args.graph is not None else int(self.world > 1)
        rows = []
        p = self.world
        for k in range(11):
            L = (1024 << (2 * k)) * 8 // b
            if 8 * L * 3 > 60e9:   # three sets of fp32 in/out: stay well inside HBM
                break
            numels = [L]
            steps = max(5, min(args.steps, int(2e9 / (8 * L)) + 5))
            rr = self.measure(e, m, numels, None, transport, want_graph, steps, 3, 3)
            del rr["sets"], rr["host"]
            T, pb = aps.layout(p, e, m, numels)
            row = {"packed_bytes": pb, "elements": L, "sync_us": round(rr["ms"] * 1e3, 2),
                   "per_rank_GBps_fp32eq": round(4 * L / (rr["ms"] * 1e-3) / 1e9, 2)}
            if p > 1:
                t_ar = rr["phase_ms"][2]
                bus = 2 * (p - 1) / p * pb / (t_ar * 1e-3) / 1e9
                row.update({"allreduce_us": round(t_ar * 1e3, 2), "busBW_GBps": round(bus, 1),
                            "busBW_frac_measured": round(bus / NVLINK_MEASURED, 4)})
                if self.comm is not None:
                    ref = {}
                    for nm_, dt, nb in (("fp32", torch.float32, 4), ("fp16", torch.float16, 2)):
                        x = torch.ones(L, dtype=dt, device=self.dev)
                        for _ in range(3):
                            self.dist.all_reduce(x)
                        torch.cuda.synchronize()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(torch.cuda.current_stream())
                        for _ in range(steps):
                            self.dist.all_reduce(x)
                        e1.record(torch.cuda.current_stream())
                        torch.cuda.synchronize()
                        t = self.max_over_ranks(e0.elapsed_time(e1) / steps)
                        ref[f"nccl_allreduce_{nm_}_us"] = round(t * 1e3, 2)
                        del x
                    row.update(ref)
            rows.append(row)
        cross = next((r["packed_bytes"] for r in rows if r.get("busBW_frac_measured", 0) >= 0.7), None)
        res = {"metric": METRIC, "value": rows[-1]["per_rank_GBps_fp32eq"] * p, "unit": UNIT, "n_gpus": p,
               "steps": args.steps, "warmup": 3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": "f32", "data": "synthetic", "ms_per_step": rows[-1]["sync_us"] / 1e3,
               "config": {"workload": "c5_message_size_sweep", "format": f"1/{e}/{m}", "transport": transport,
                          "parallelism": f"dp{p}"},
               "sweep": rows, "busBW_70pct_crossover_packed_bytes": cross}
        if self.rank == 0:
            print(json.dumps(res), flush=True)
        self.close()

    def close(self):
        if self.comm:
            self.aps.nccl_comm_destroy(self.comm)
            self.comm = None
        if self.dist:
            self.dist.destroy_process_group()


def format_runs(numels, fmts, p, rank):
    """Per reduce-scatter step of `rank`: the number of format runs in the chunk
    it receives (one reduce launch each; padding tiles take the last format)."""
    tile_fmt = []
    for n, f in zip(numels, fmts):
        tile_fmt += [f] * ((n + 127) // 128)
    Tp = (len(tile_fmt) + p - 1) // p * p
    tile_fmt += [fmts[-1]] * (Tp - len(tile_fmt))
    ct = Tp // p
    out = []
    for s in range(p - 1):
        rc = (rank - 2 - s) % p
        seg = tile_fmt[rc * ct:(rc + 1) * ct]
        out.append(1 + sum(1 for a, b in zip(seg, seg[1:]) if a != b))
    return out


def main():
    args = parse()
    world, _, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    b = Bench(args)
    if args.config == "c5":
        b.run_c5()
    else:
        b.run()


if __name__ == "__main__":
    main()
