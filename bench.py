"""Benchmark of the PQ / IVF hot path on B200 (contract: one JSON line).

Workload (N=1): BASELINE.json configs[1] -- N=1,000,000 x D=128 fp32 rows of a
seeded 256-component Gaussian mixture; PQ k-means (25 iterations on a seeded
100k-row sample) then encode of all 1M rows.  The headline `value` is PQ
encode vectors/s at M=8, Ks=256 (the reference's own config-1 codebook shape);
the sweep over M in {4,8,16,32} x Ks in {16,64,256}, the k-means iterations/s
and the config-3 ADC search queries/s (1M items, nlist 1024, 10k queries,
nprobe 16, k 10) ride along in the same line.

A step = one pq_encode of the 1M device-resident rows (512 MB > the 126 MB
L2, so no flush is needed between steps).  `e2e` is the same metric through
the C ABI with pinned HOST buffers (H2D of the rows and D2H of the codes in
the timed region).  `--impl reference` times the reference's own pq_encode
(oracle/_ref, compiled from its sources) on the host cores.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PQ encode vectors/s and k-means iters/s at M,Ks; ADC queries/s; % of roofline"
N_ROWS = 1_000_000
DIMS = 128
COMPONENTS = 256
SAMPLE = 100_000
FIT_ITERS = 25
HEAD_M, HEAD_KS = 8, 256
SEED = 2604


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed over NCCL, one process per GPU)
# ---------------------------------------------------------------------------
def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "RANK" in os.environ:  # launched by torchrun (any world size): NCCL process group
        # keep stdout to the one JSON line: NCCL's own log (version banner at
        # NCCL_DEBUG >= VERSION, INFO lines) goes to stderr
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def distributed():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def barrier(world):
    if distributed():
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if not distributed():
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled every 100 ms through NVML while
    the timed region runs (the recipe's clocks line)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(self.device)).split(",")[self.device]) \
                if os.environ.get("CUDA_VISIBLE_DEVICES") else self.device
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: report no samples rather than fail
            log("clock sampler unavailable:", e)
            self.nv = None
        return self

    def _sample(self):
        try:
            mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
            rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append((mhz, rs))
        except Exception:
            pass

    def _run(self):
        while not self.stop.is_set():
            self._sample()
            self.stop.wait(0.005)

    def __exit__(self, *exc):
        self.stop.set()
        if getattr(self, "t", None):
            self.t.join(timeout=2)
        if self.nv is not None:
            self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set()
        for _, rs in self.samples:
            for name, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": float(np.median([m for m, _ in self.samples])),
                "sm_max_mhz": float(self.max_mhz), "reasons": sorted(reasons),
                "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic(kernel_key: str):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(kernel_key, {})
    return v.get("dram_bytes_per_launch")


# ---------------------------------------------------------------------------
# reference arm (the reference's own CPU code, all host threads)
# ---------------------------------------------------------------------------
def reference_encode_rate(x: np.ndarray, tables: np.ndarray, threads: int, rows: int):
    import oracle
    R = oracle.ref_impl()
    sample = np.ascontiguousarray(x[:rows])
    t0 = time.perf_counter()
    R.pq_encode(sample, tables, threads=threads)
    dt = time.perf_counter() - t0
    return rows / dt, dt


def rank_of() -> int:
    return int(os.environ.get("RANK", "0"))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


def cpu_baselines(x_host, train_h, adc_host, budget_s: float = 25.0):
    """The reference (oracle/_ref, compiled from its sources) on this host's
    cores, on bounded samples of the bench's own workloads:
    k-means passes of pq_fit (1 thread; all cores = one thread per subspace,
    kmeans_fit's documented concurrency, kmeans.hpp:40) and ivf_query over the
    configs[2] index the GPU built (1 thread; all cores = queries split over
    threads, a frozen index is reader-safe, ivf.hpp:20-22)."""
    import oracle
    R = oracle.ref_impl()
    thr = max(1, R.hardware_concurrency())
    out = {"cpu_model": cpu_model(), "threads": thr}
    ds = DIMS // HEAD_M
    # k-means: 2 passes (1 update) of the headline pq_fit on the 100k sample
    t0 = time.perf_counter()
    R.kmeans_fit(np.ascontiguousarray(train_h[:, :ds]), HEAD_KS, 2, SEED, 0.0)
    one = time.perf_counter() - t0
    t0 = time.perf_counter()
    R.pq_fit_stats(train_h, HEAD_M, HEAD_KS, 2, SEED, thr)
    allc = time.perf_counter() - t0
    # per full iteration over all M subspaces (2 passes per fit measured)
    out["kmeans_iters_per_s_1thread"] = 2.0 / (one * HEAD_M)
    out["kmeans_iters_per_s_allcores"] = 2.0 / allc
    out["kmeans_sample"] = (f"kmeans_fit 2 passes of one subspace (100k x {ds}, Ks={HEAD_KS}) x M={HEAD_M} "
                            f"on 1 thread; pq_fit 2 passes with the M subspaces on {thr} threads")
    if adc_host is not None:
        a = adc_host
        ids = np.arange(a["codes"].shape[0], dtype=np.uint64)
        idx = R.ivf_build_with_centroids_mt(a["codes"], ids, a["tables"], a["coarse"], thr)
        q = a["queries"]
        n1 = 300
        t0 = time.perf_counter()
        idx.query_batch(q[:n1], a["k"], a["nprobe"], threads=1)
        q1 = n1 / (time.perf_counter() - t0)
        nall = min(q.shape[0], max(n1, int(q1 * thr * 2)))
        t0 = time.perf_counter()
        idx.query_batch(q[:nall], a["k"], a["nprobe"], threads=thr)
        qa = nall / (time.perf_counter() - t0)
        out["adc_queries_per_s_1thread"] = q1
        out["adc_queries_per_s_allcores"] = qa
        out["adc_sample"] = (f"ivf_query (nprobe {a['nprobe']}, k {a['k']}) over the configs[2] index "
                             f"(1M items, nlist 1024): {n1} queries on 1 thread, {nall} on {thr} threads")
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    from paper_2604_21645_b200.datagen import gaussian_mixture
    if not oracle.ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libpqii_ref.so not built"})
        return
    R = oracle.ref_impl()
    threads = max(1, R.hardware_concurrency())
    x = gaussian_mixture(N_ROWS, DIMS, COMPONENTS, SEED)
    tables = reference_codebook(x)
    rows = min(N_ROWS, 2500 * threads)  # ~0.1-0.2 s per step at ~20k vec/s/thread
    for _ in range(args.warmup):
        reference_encode_rate(x, tables, threads, rows)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        reference_encode_rate(x, tables, threads, rows)
    dt = (time.perf_counter() - t0) / args.steps
    v = rows / dt
    emit({
        "metric": METRIC, "value": v, "unit": "vectors/s", "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(world),
        "cpu_baseline": {"value": v, "unit": "vectors/s", "cores": threads, "kind": "reference",
                         "sample": f"pq_encode of {rows} of the 1M rows per step, M={HEAD_M} Ks={HEAD_KS}, "
                                   f"chunk_rows over {threads} threads (proj/src/pipeline.cpp:226-231)"},
        "e2e": {"value": v, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


def reference_codebook(x):
    """A fixed M=8, Ks=256 codebook for the reference arm: rows of the sample
    (fitting it on the CPU would take minutes; encode cost does not depend on
    the codebook values)."""
    from paper_2604_21645_b200.datagen import strided_sample
    s = strided_sample(N_ROWS, SAMPLE, SEED)
    ds = DIMS // HEAD_M
    t = np.empty((HEAD_M, HEAD_KS, ds), np.float32)
    for m in range(HEAD_M):
        t[m] = x[s[m * HEAD_KS:(m + 1) * HEAD_KS], m * ds:(m + 1) * ds]
    return t


def config_block(world):
    return {"workload": "BASELINE configs[1]: 1M x 128 fp32, 256-comp Gaussian mixture; "
                        f"PQ fit {FIT_ITERS} iters on seeded 100k sample + encode all rows "
                        f"(headline M={HEAD_M}, Ks={HEAD_KS}); ADC per configs[2]",
            "rows_per_gpu": N_ROWS, "dims": DIMS, "M": HEAD_M, "Ks": HEAD_KS,
            "global_rows": N_ROWS * world, "parallelism": f"row shards x{world}",
            "l2": "inputs (512 MB/GPU) exceed the 126 MB L2; no flush needed",
            "seed": SEED}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local):
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture, strided_sample

    torch.cuda.set_device(local)
    ctx = pqii.Context(local)
    # a dedicated stream shared by torch (events, copies) and libpqg (kernels);
    # torch's legacy default stream has handle 0, which the C ABI reads as
    # "use the context's own stream", so it cannot be used here
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    vp = C.c_void_p

    # per-rank shard of rows (weak scaling: 1M rows per GPU), generated per shard
    x_host = gaussian_mixture(N_ROWS, DIMS, COMPONENTS, SEED, stream=2 + rank)
    x = torch.from_numpy(x_host).cuda()
    sample_idx = torch.from_numpy(strided_sample(N_ROWS, SAMPLE, SEED)).cuda()
    train = x.index_select(0, sample_idx).contiguous()

    def fit(M, ks, iters=FIT_ITERS):
        ds = DIMS // M
        tables = torch.empty((M, ks, ds), dtype=torch.float32, device="cuda")
        it = np.zeros(M, np.uint32)
        L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), SAMPLE, DIMS, M, ks, iters, SEED,
                               vp(tables.data_ptr()), it.ctypes.data_as(vp), None), "pq_fit")
        return tables, int(it.max())

    def encode(tables, M, ks, codes):
        L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), N_ROWS, M, ks, DIMS // M,
                                  vp(tables.data_ptr()), vp(codes.data_ptr())), "encode")

    def rmse_of(tables, M, ks, codes):
        sse = C.c_double()
        L.check(lib.pqg_pq_recon_sse(ctx.h, vp(x.data_ptr()), vp(codes.data_ptr()), N_ROWS, M, ks,
                                     DIMS // M, vp(tables.data_ptr()), C.byref(sse)), "sse")
        return (sse.value / (N_ROWS * DIMS)) ** 0.5

    def timed(fn, steps, warmup, region=None):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        # --profile-region NAME: only this timed region is visible to a
        # profiler started with `ncu --profile-from-start off`
        prof = region is not None and region == args.profile_region
        if prof:
            torch.cuda.cudart().cudaProfilerStart()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        if prof:
            torch.cuda.cudart().cudaProfilerStop()
        barrier(world)
        return max_over_ranks(a.elapsed_time(b) / steps, world)

    # ---- k-means fit at the headline point (iters/s)
    fit(HEAD_M, HEAD_KS)  # warm-up (also JIT of module-level state)
    torch.cuda.synchronize()
    if args.profile_region == "fit":
        torch.cuda.cudart().cudaProfilerStart()
    t0 = time.perf_counter()
    tables, iters_run = fit(HEAD_M, HEAD_KS)
    torch.cuda.synchronize()
    if args.profile_region == "fit":
        torch.cuda.cudart().cudaProfilerStop()
    fit_s = max_over_ranks(time.perf_counter() - t0, world)
    kmeans_ips = iters_run / fit_s

    # ---- exact sharded PQ fit over the ranks' samples (the north-star
    # exchange: one all-reduce of sums / counts / exponent ranges per
    # iteration over NCCL; a 1-rank NCCL group when not under torchrun)
    sharded_fit = None
    if not args.quick:
        from paper_2604_21645_b200 import dist as D
        if not distributed():
            import torch.distributed as tdist
            tdist.init_process_group("nccl", store=tdist.HashStore(), rank=0, world_size=1,
                                     device_id=torch.device("cuda", local))
        comm, be = D.Comm(), D.CudaBackend(local)
        be.ctx.set_stream(stream.cuda_stream)
        ds = DIMS // HEAD_M
        seeds = [SEED + m for m in range(HEAD_M)]
        D.kmeans_fit_sharded(comm, be, train, HEAD_M, ds, ds, HEAD_KS, 2, seeds)  # warm-up
        torch.cuda.synchronize()
        barrier(world)
        st = {}
        t0 = time.perf_counter()
        sf = D.kmeans_fit_sharded(comm, be, train, HEAD_M, ds, ds, HEAD_KS, FIT_ITERS, seeds, 1e-4, stats=st,
                                  force_exchange=True)
        torch.cuda.synchronize()
        sf_s = max_over_ranks(time.perf_counter() - t0, world)
        # the default path (a 1-rank group runs the single-process fit)
        st_def = {}
        t0 = time.perf_counter()
        D.kmeans_fit_sharded(comm, be, train, HEAD_M, ds, ds, HEAD_KS, FIT_ITERS, seeds, 1e-4, stats=st_def)
        torch.cuda.synchronize()
        sf_def_s = max_over_ranks(time.perf_counter() - t0, world)
        same = bool(torch.equal(sf.tables, tables)) if world == 1 else None
        # the same protocol with the loop in C++ and NCCL issued by the library
        # (pqg_kmeans_fit_sharded, csrc/kmnccl.cu), exchange always run
        native = None
        try:
            nc = D.NcclComm(comm, be)
            try:
                D.kmeans_fit_sharded_native(nc, train, HEAD_M, ds, ds, HEAD_KS, 2, seeds)  # warm-up
                torch.cuda.synchronize()
                barrier(world)
                stn = {}
                t0 = time.perf_counter()
                sfn = D.kmeans_fit_sharded_native(nc, train, HEAD_M, ds, ds, HEAD_KS, FIT_ITERS, seeds, 1e-4,
                                                  stats=stn)
                torch.cuda.synchronize()
                nat_s = max_over_ranks(time.perf_counter() - t0, world)
                native = {"seconds": nat_s, "iters_per_s": int(np.max(sfn.iterations_run)) / nat_s,
                          "host": stn.get("host"), "replay_columns": stn.get("replay_columns"),
                          "bit_identical_to_single_process":
                              bool(torch.equal(sfn.tables, tables)) if world == 1 else None}
            finally:
                nc.close()
        except Exception as e:  # NCCL unavailable: reported, not fatal
            native = {"unavailable": str(e)[:200]}
        sharded_fit = {"global_sample_rows": SAMPLE * world, "iters_run": int(np.max(sf.iterations_run)),
                       "seconds": sf_s, "iters_per_s": int(np.max(sf.iterations_run)) / sf_s,
                       "single_process_seconds": fit_s,
                       "exchange_forced": True,
                       "default_path_seconds": sf_def_s,
                       "default_path": st_def.get("path", "exchange"),
                       "allreduce_bytes_per_iter": st["allreduce_bytes"] / max(1, st["iterations"]),
                       "replay_columns": st["replay_columns"], "reseeds": st["reseeds"],
                       "replay": st.get("replay"),
                       "chain_bytes_per_iter": st.get("chain_bytes", 0) / max(1, st["iterations"]),
                       "allgather_bytes_per_iter": st.get("allgather_bytes", 0) / max(1, st["iterations"]),
                       "bit_identical_to_single_process": same,
                       "native_host": native}

    # ---- headline encode, timed with profiling of the dominant kernel
    codes = torch.empty((N_ROWS, HEAD_M), dtype=torch.uint8, device="cuda")
    encode(tables, HEAD_M, HEAD_KS, codes)
    l0 = ctx.launches
    with ClockSampler(local) as clk:
        ctx.profile(True)
        ms = timed(lambda: encode(tables, HEAD_M, HEAD_KS, codes), args.steps, args.warmup, "encode")
        n_near, near_ms = ctx.profile_read("nearest_tc")
        screen_kernel = "umma_screen (tcgen05 3xTF32, TMEM accumulator)"
        if n_near == 0:
            n_near, near_ms = ctx.profile_read("nearest")
            screen_kernel = "nearest_kernel (FP32 FFMA screen)"
        n_fix, fix_ms = ctx.profile_read("fixup")
        n_norm, norm_ms = ctx.profile_read("norms")
        ctx.profile(False)
    launches_per_step = (ctx.launches - l0) / (args.steps + args.warmup)
    value = N_ROWS * world / (ms / 1e3)
    head_rmse = rmse_of(tables, HEAD_M, HEAD_KS, codes)

    # roofline of the dominant kernel (fp32 screen; 2*Ks*D flops per vector)
    peaks, src = measured_peaks()
    near_avg_ms = near_ms / max(n_near, 1)
    flops_per_launch = float(N_ROWS) * 2 * HEAD_KS * DIMS
    achieved_tflops = flops_per_launch / (near_avg_ms / 1e3) / 1e12
    props = torch.cuda.get_device_properties(local)
    fp32_nominal = props.multi_processor_count * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    probe = C.c_double()
    L.check(lib.pqg_fp32_probe(ctx.h, C.byref(probe)), "fp32_probe")
    fp32_peak = float(probe.value)
    traffic = ncu_traffic("prof_enc_r2h")
    tc_bf16 = float(peaks.get("bf16_tflops", 1590.0))
    psrc_tc = src
    tc_peak = tc_bf16 / 2.0 / 3.0

    # ---- e2e through the C ABI with pinned host buffers
    xh = torch.from_numpy(x_host).pin_memory()
    ch = torch.empty((N_ROWS, HEAD_M), dtype=torch.uint8).pin_memory()
    tables_h = tables.cpu().contiguous()

    def e2e_step():
        L.check(lib.pqg_pq_encode(ctx.h, vp(xh.data_ptr()), N_ROWS, HEAD_M, HEAD_KS, DIMS // HEAD_M,
                                  vp(tables_h.data_ptr()), vp(ch.data_ptr())), "encode_e2e")

    for _ in range(args.warmup):
        e2e_step()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps, world)
    assert torch.equal(ch, codes.cpu()), "e2e codes differ from the device-resident run"

    # ---- sweep over M x Ks (configs[1]) -- encode vec/s and RMSE per point
    sweep = []
    if not args.quick:
        for M in (4, 8, 16, 32):
            for ks in (16, 64, 256):
                t, itr = fit(M, ks)
                cds = torch.empty((N_ROWS, M), dtype=torch.uint8, device="cuda")
                ms_pt = timed(lambda: encode(t, M, ks, cds), max(2, args.steps // 2), 1)
                vps = N_ROWS * world / (ms_pt / 1e3)
                fl = 2.0 * ks * DIMS
                by = 4.0 * DIMS + M
                bound_s = max(fl / (fp32_peak * 1e12), by / (peaks["hbm_gbs"] * 1e9))
                sweep.append({"M": M, "Ks": ks, "encode_vectors_per_s": vps,
                              "rmse": rmse_of(t, M, ks, cds), "fit_iters_run": itr,
                              "roofline_vectors_per_s": 1.0 / bound_s,
                              "frac": vps / world * bound_s})
                del cds

    # ---- configs[2]: ADC search queries/s
    adc = None
    if not args.quick:
        adc = adc_bench(ctx, lib, L, x, train, args, world, stream, timed)

    # ---- CPU baseline: the compiled reference on this host (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            import oracle
            if oracle.ref_available():
                R = oracle.ref_impl()
                thr = max(1, R.hardware_concurrency())
                rows = min(N_ROWS, 4000 * thr)
                v_cpu, dt = reference_encode_rate(x_host, tables_h.numpy(), thr, rows)
                reps = max(1, int(10.0 / max(dt, 1e-3)))
                reps = min(reps, 20)
                tot = 0.0
                for _ in range(reps):
                    _, d1 = reference_encode_rate(x_host, tables_h.numpy(), thr, rows)
                    tot += d1
                v_cpu = rows * reps / tot
                cpu = {"value": v_cpu, "unit": "vectors/s", "cores": thr, "kind": "reference",
                       "sample": f"{reps} x pq_encode of {rows} rows (M={HEAD_M}, Ks={HEAD_KS}) "
                                 f"with chunk_rows over {thr} threads; reference compiled -O3"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "vectors/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank != 0:
        return
    adc_host = adc.pop("_host", None) if adc else None
    if cpu is not None and cpu.get("value") and not args.no_cpu:
        try:
            cpu["extra"] = cpu_baselines(x_host, train.cpu().numpy(), adc_host)
        except Exception as e:  # reported, never required
            cpu["extra"] = {"unavailable": str(e)}
    out = {
        "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian mixture, BASELINE configs[1]/[2] shapes)",
        "config": config_block(world),
        "rmse": head_rmse,
        "kmeans_iters_per_s": kmeans_ips,
        # one iteration = one assignment pass over the sample (2*N*Ks*D flop, the
        # SURVEY 8(d) K1 count) plus the mean update; FP32 peak as for the encode
        "kmeans_roofline": {"bound": "fp32",
                            "achieved": 2.0 * SAMPLE * HEAD_KS * DIMS * kmeans_ips / 1e12,
                            "peak": fp32_peak, "unit": "TFLOP/s",
                            "frac": 2.0 * SAMPLE * HEAD_KS * DIMS * kmeans_ips / 1e12 / fp32_peak,
                            "algorithmic": "2*N*Ks*D flop per iteration, N = sample rows"},
        "kmeans_fit": {"M": HEAD_M, "Ks": HEAD_KS, "sample_rows": SAMPLE, "iters_run": iters_run,
                       "seconds": fit_s},
        "sharded_pq_fit": sharded_fit,
        "adc": adc,
        "sweep": sweep,
        # the screen's products run on the tensor pipe as 3xTF32 (three tf32
        # products per fp32-accurate product): its roof is the dense TF32 rate
        # (half the measured bf16 GEMM rate) / 3.  roofline_fp32 is the
        # north star's definition (FP32 FFMA peak), which the tensor path exceeds.
        "roofline": {"bound": "tensor", "achieved": achieved_tflops, "peak": tc_peak,
                     "unit": "TFLOP/s", "frac": achieved_tflops / tc_peak, "traffic": traffic,
                     "kernel": screen_kernel,
                     "algorithmic": "2*Ks*D = 65536 flop per vector x 1M vectors per launch",
                     "peak_source": f"{psrc_tc}: bf16_tflops {tc_bf16:.1f} / 2 (tf32 dense) / 3 (3xTF32 split)",
                     "fp32_nominal_tflops": fp32_nominal,
                     "kernel_ms": near_avg_ms, "launches": n_near,
                     # profiling spans warm-up + timed steps: one launch of each per step
                     "share_of_step": near_avg_ms / max(ms, 1e-9),
                     "fixup_ms_per_step": fix_ms / max(n_fix, 1),
                     "norms_ms_per_step": norm_ms / max(n_norm, 1)},
        "roofline_fp32": {"bound": "fp32", "achieved": achieved_tflops, "peak": fp32_peak, "unit": "TFLOP/s",
                          "frac": achieved_tflops / fp32_peak,
                          "peak_source": "measured: register-operand FFMA probe (pqg_fp32_probe) on this GPU"},
        "cpu_baseline": cpu,
        "e2e": {"value": N_ROWS * world / e2e_s, "unit": "vectors/s",
                "h2d_bytes_per_step": N_ROWS * DIMS * 4 + HEAD_M * HEAD_KS * (DIMS // HEAD_M) * 4,
                "d2h_bytes_per_step": N_ROWS * HEAD_M,
                "path": "pqg_pq_encode with pinned host input/output (C ABI)"},
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "clocks": clk.summary(),
    }
    emit(out)


def adc_bench(ctx, lib, L, x, train, args, world, stream, timed):
    """configs[2]: M=16, Ks=256, nlist=1024 coarse centroids fitted on the 100k
    sample, coarse-assign + CSR of all rows, 10k queries, nprobe 16, k 10."""
    import torch
    from paper_2604_21645_b200.datagen import gaussian_mixture
    vp = C.c_void_p
    M, ks, nlist, nq, nprobe, k = 16, 256, 1024, 10_000, 16, 10
    tables = torch.empty((M, ks, DIMS // M), dtype=torch.float32, device="cuda")
    L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), SAMPLE, DIMS, M, ks, 20, SEED,
                           vp(tables.data_ptr()), None, None))
    coarse = torch.empty((nlist, DIMS), dtype=torch.float32, device="cuda")
    inertia = C.c_double()
    it = C.c_uint32()
    for rep in range(2):  # the second (warm) fit is timed
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.check(lib.pqg_kmeans_fit(ctx.h, vp(train.data_ptr()), SAMPLE, DIMS, nlist, 20, SEED + M,
                                   1e-4, vp(coarse.data_ptr()), None, C.byref(inertia), C.byref(it),
                                   None))
        torch.cuda.synchronize()
        coarse_s = time.perf_counter() - t0
    codes = torch.empty((N_ROWS, M), dtype=torch.uint8, device="cuda")
    L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), N_ROWS, M, ks, DIMS // M,
                              vp(tables.data_ptr()), vp(codes.data_ptr())))
    ids = torch.arange(N_ROWS, dtype=torch.int64, device="cuda") + int(os.environ.get("RANK", "0")) * N_ROWS
    h = C.c_void_p()
    for rep in range(2):  # the second (warm) build is timed
        if rep:
            lib.pqg_index_destroy(h)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.check(lib.pqg_ivf_build_with_centroids(ctx.h, vp(tables.data_ptr()), M, ks, DIMS // M,
                                                 vp(codes.data_ptr()), vp(ids.data_ptr()), N_ROWS,
                                                 vp(coarse.data_ptr()), nlist, C.byref(h)))
        torch.cuda.synchronize()
        build_s = time.perf_counter() - t0
    q = torch.from_numpy(gaussian_mixture(nq, DIMS, COMPONENTS, SEED, stream=1)).cuda()
    oi = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    od = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    oc = torch.empty((nq,), dtype=torch.int32, device="cuda")

    if distributed():
        # every rank searches its shard (global ids rank*N + i), then the
        # per-shard top-k lists are all-gathered and merged by (dist, id)
        import torch.distributed as dist
        gi = torch.empty((world, nq, k), dtype=torch.int64, device="cuda")
        gd = torch.empty((world, nq, k), dtype=torch.float64, device="cuda")
        gc = torch.empty((world, nq), dtype=torch.int32, device="cuda")
        mi = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        md = torch.empty((nq, k), dtype=torch.float64, device="cuda")
        mc = torch.empty((nq,), dtype=torch.int32, device="cuda")

    def search():
        L.check(lib.pqg_index_search(ctx.h, h, vp(q.data_ptr()), nq, k, nprobe, 0, 0.0,
                                     vp(oi.data_ptr()), vp(od.data_ptr()), vp(oc.data_ptr())))
        if distributed():
            dist.all_gather_into_tensor(gi, oi)
            dist.all_gather_into_tensor(gd, od)
            dist.all_gather_into_tensor(gc, oc)
            L.check(lib.pqg_topk_merge(ctx.h, vp(gi.data_ptr()), vp(gd.data_ptr()), vp(gc.data_ptr()),
                                       world, nq, k, vp(mi.data_ptr()), vp(md.data_ptr()), vp(mc.data_ptr())))

    ctx.profile(True)
    ms = timed(search, max(3, args.steps // 2), 2, "adc")
    n_scan, scan_ms = ctx.profile_read("adc_scan")
    n_sel, sel_ms = ctx.profile_read("probe_select")
    n_mat, mat_ms = ctx.profile_read("distance_matrix")
    n_mtc, mtc_ms = ctx.profile_read("distance_matrix_tc")
    n_spl, spl_ms = ctx.profile_read("big_split")
    ctx.profile(False)
    off = torch.empty(nlist + 1, dtype=torch.int64)
    L.check(lib.pqg_index_export(ctx.h, h, vp(off.data_ptr()), None, None, None, None))
    # candidates actually scanned: S_q = sum of the probed lists' lengths
    probes = torch.empty((nq, nprobe), dtype=torch.int32, device="cuda")
    L.check(lib.pqg_index_probe(ctx.h, h, vp(q.data_ptr()), nq, nprobe, vp(probes.data_ptr())))
    sizes = (off[1:] - off[:-1]).cuda()
    cand = int(sizes[probes.long()].sum())
    host_arrays = None
    if rank_of() == 0 and world == 1:  # for the CPU baseline leg (reference on the same index)
        host_arrays = {"codes": codes.cpu().numpy(), "coarse": coarse.cpu().numpy(),
                       "tables": tables.cpu().numpy(), "queries": q.cpu().numpy(),
                       "nprobe": nprobe, "k": k}
    lib.pqg_index_destroy(h)
    scan_ms_b = scan_ms / (max(3, args.steps // 2) + 2)
    peaks, psrc = measured_peaks()
    code_bytes = cand * M  # algorithmic bytes: the probed lists' code rows, read once
    ach = code_bytes / (scan_ms_b / 1e3) / 1e9
    return {"_host": host_arrays, "queries_per_s": nq / (ms / 1e3), "ms_per_batch": ms, "nq": nq,
            "candidates_per_query": cand / nq,
            # the 16 MB of codes stay L2-resident, so the scan is
            # also reported against the shared-memory LUT-gather bound (one
            # 4-byte LDS per (candidate, subspace); 32 per clock per SM)
            "roofline_lut": {"bound": "smem_lut", "unit": "G lookups/s",
                             "achieved": cand * M / (scan_ms_b / 1e3) / 1e9,
                             "peak": 32 * 148 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e9,
                             "frac": (cand * M / (scan_ms_b / 1e3)) /
                                     (32 * 148 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6)},
            "roofline_scan": {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                              "unit": "GB/s", "frac": ach / peaks["hbm_gbs"],
                              "kernel": "adc_scan_kernel", "kernel_ms": scan_ms_b,
                              "algorithmic": "S_q*M code bytes per query (S_q measured from the "
                                             "probe lists) x nq per launch",
                              "peak_source": psrc,
                              "note": "the 16 MB of codes are L2-resident across the batch; "
                                      "the scan is bound by shared-memory LUT gathers"},
            "index_rows": N_ROWS * world, "shards": world,
            "nprobe": nprobe, "k": k, "nlist": nlist, "M": M, "Ks": ks,
            "coarse_kmeans_seconds": coarse_s, "coarse_iters_run": it.value,
            "ivf_build_seconds": build_s,
            "kernel_ms_per_batch": {k_: v_ / (max(3, args.steps // 2) + 2) for k_, v_ in
                                    (("adc_scan", scan_ms), ("probe_select", sel_ms),
                                     ("distance_matrix_fp32", mat_ms),
                                     ("distance_matrix_tc", mtc_ms), ("operand_split", spl_ms))},
            "max_list": int((off[1:] - off[:-1]).max())}


_JSON_FD = None


def emit(obj):
    """The one JSON line, written to the process's original stdout."""
    line = (json.dumps(obj) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line)


def main():
    global _JSON_FD
    # everything else written to fd 1 (library banners such as NCCL's version
    # line, printed from C at communicator init) goes to stderr
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true", help="headline only (no sweep / ADC)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--profile-region", default=None, choices=[None, "encode", "adc", "fit"],
                    help="bracket this timed region with cudaProfilerStart/Stop (ncu --profile-from-start off)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "RANK" not in os.environ and args.impl == "ours":
        # one process per GPU: relaunch under torchrun (the driver launches it
        # that way itself); the JSON line comes from rank 0's stdout
        import socket
        import subprocess
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        os.dup2(_JSON_FD, 1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world)
        return
    rank, world, local = dist_setup()
    run_ours(args, rank, world, local)
    if distributed():
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
