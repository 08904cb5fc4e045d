#!/usr/bin/env python
"""QFT quantized Lion step throughput on LLaMA-2-7B-shaped model state (BASELINE.json).

Own arm (default):
  python bench.py [--gpus N --steps K --warmup W]
  One "step" = one fused quantized Lion step over every weight tensor of the model
  (lion_step_quantized, optimizer.hpp:85-120): dequant g,m,w -> Lion -> requant m
  (fresh params) -> requant w (cached thresholds) + CSR re-extraction, reference
  layout b=8, p=1% percentile outliers, u8 gradient codes (the GradientStack entry).
  Synthetic weights/gradients generated on the device (deterministic generator,
  bit-identical to oracle/synth.c); inputs larger than L2 (34.8 GB per step).
Reference arm:
  python bench.py --impl reference ...
  the reference's own CPU implementation (oracle/_ref: the reference headers
  compiled unmodified) on the host cores, bounded sample of the same workload.

Prints ONE JSON line (rank 0).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QFT Lion step Gparams/s + HBM GB/s vs peak, LLaMA-2-7B, 1/2/4/8 B200"
UNIT = "Gparams/s"
BIT_WIDTH = 8
FRACTION = 0.01
HYPER = dict(lr=2e-5, beta1=0.9, beta2=0.99, weight_decay=0.0)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index=0):
        self.samples, self.proc, self.index = [], None, index

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm, smax = [], []
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                smax.append(float(s[1]))
            except ValueError:
                continue
            for n, v in zip(names, s[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU arm
def host_cpu():
    """(usable host threads, CPU model) of this box"""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return n, model


def layer_row_chunks(rows_per_chunk=512):
    """One LLaMA-2-7B decoder layer's weight matrices (4 x 4096x4096, 2 x 11008x4096,
    4096x11008; 202.4 M params) cut into row blocks of <= rows_per_chunk rows.  The step is
    per row (optimizer.hpp:103-118), so a row block stepped as its own layer is the same
    work and the same bytes; the blocks let every host thread stay busy to the end."""
    mats = [(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)]
    out = []
    for r, c in mats:
        for r0 in range(0, r, rows_per_chunk):
            out.append((min(rows_per_chunk, r - r0), c))
    return out


def cpu_reference_run(steps, warmup, threads=None, sample=None):
    """Time qft::lion_step_quantized (the unmodified reference, compiled from its headers)
    on the host cores: a bounded sample of the 7B workload -- one decoder layer's matrices
    in row blocks, several times more blocks than threads, handed out longest-first."""
    from oracle import oracle as O
    if not O.available("reference"):
        O.build()
    lib = C.CDLL(O.REF_LIB)
    lib.qr_bench_create.restype = C.c_void_p
    lib.qr_bench_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_uint64,
                                    C.c_int, C.c_double, C.c_float, C.c_float, C.c_float,
                                    C.c_float, C.c_int]
    lib.qr_bench_step.restype = C.c_double
    lib.qr_bench_step.argtypes = [C.c_void_p, C.c_int]
    lib.qr_bench_params.restype = C.c_int64
    lib.qr_bench_params.argtypes = [C.c_void_p]
    lib.qr_bench_destroy.argtypes = [C.c_void_p]
    ncpu, model = host_cpu()
    sample = sample or layer_row_chunks()
    threads = min(threads or ncpu, len(sample))   # the threads that actually run
    rows = (C.c_int * len(sample))(*[r for r, _ in sample])
    cols = (C.c_int * len(sample))(*[c for _, c in sample])
    h = lib.qr_bench_create(len(sample), rows, cols, 1234, BIT_WIDTH, FRACTION, HYPER["lr"],
                            HYPER["beta1"], HYPER["beta2"], HYPER["weight_decay"], threads)
    n = lib.qr_bench_params(h)
    for _ in range(warmup):
        lib.qr_bench_step(h, threads)
    ts = [lib.qr_bench_step(h, threads) for _ in range(steps)]
    lib.qr_bench_destroy(h)
    t = statistics.median(ts)
    return {"value": n / t / 1e9, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"one LLaMA-2-7B decoder layer's 7 weight matrices ({n / 1e6:.1f} M params) "
                      f"in {len(sample)} row blocks of <= 512 rows, b=8 p=1% u8 gradient codes, "
                      f"median of {steps} steps; {threads} host threads (dynamic, longest "
                      f"block first) of {ncpu} usable on '{model}'",
            "cpu_model": model, "host_threads_usable": ncpu,
            "ms_per_step": t * 1e3, "params": n}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    steps = max(1, min(args.steps, 3))
    warm = min(args.warmup, 1)
    cb = cpu_reference_run(steps, warm)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
        "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": cb["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": "llama2-7b-shaped quantized Lion step (bounded CPU sample)",
                   "bit_width": BIT_WIDTH, "outlier_fraction": FRACTION},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                            "cpu_model")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def build_state(shapes, q, seed_base=1234):
    import torch
    st = q.QftModelState(shapes, bit_width=BIT_WIDTH, grad_kind="u8")
    st.init_from_weights(lambda i: q.synth(shapes[i], seed_base + i, 0.02, 0.005),
                         FRACTION, "percentile")
    for i, sh in enumerate(shapes):
        g = q.synth(sh, seed_base + 100000 + i, 1e-3, 0.0)
        gq = q.quantize_state(g, BIT_WIDTH, check=False)
        c, s, z = st.grad_views(i)
        c.copy_(gq.data)
        s.copy_(gq.params.scale)
        z.copy_(gq.params.zero_point)
        del g, gq
    torch.cuda.synchronize()
    return st


def algorithmic_bytes(st, g, nnz_in, nnz_out):
    """per param 5 B (read w,m,g codes; write w,m codes) + 8 B per old
    and per new CSR entry + 48 B per row (w scale/zp/t_min/t_max, row_ptr in/out,
    m scale/zp in/out, g scale/zp)."""
    params = sum(st.shapes[i][0] * st.shapes[i][1] for i in g.members)
    return 5 * params + 8 * (nnz_in + nnz_out) + 48 * g.rows


def run_gpu_arm(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2310_07147_b200 as q
    from paper_2310_07147_b200.shapes import count, llama2_7b

    full = llama2_7b()
    if world > 1:
        return run_multi_gpu(args, full, world, rank, local, q)
    shapes = full
    t0 = time.time()
    st = build_state(shapes, q, 1234)
    setup_s = time.time() - t0
    stream = torch.cuda.current_stream()

    # warm-up (also gives the momentum real codes: m0 = LionState::init zeros)
    for _ in range(args.warmup):
        st.step(**HYPER, check=True)   # validates and re-plans CSR slots if a row grew
    nnz_before = [st.group_nnz(g) for g in st.groups]

    # ---------------- timed region: device-resident inputs ----------------
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    ms = timed_region(st, args.steps, stream, HYPER)
    clocks = clk.stop()
    st.check()  # raises on CSR overflow / degenerate rows (never silently)
    st_rows, gen_rows = st.tier_rows()
    tiers = st.tiers()
    nnz_after = [st.group_nnz(g) for g in st.groups]
    params_local, rows_local = count(shapes)
    value = params_local / (ms * 1e-3) / 1e9

    # roofline of the dominant launch: one step is ONE concurrent launch group (every
    # width class forked onto its own stream and joined back), so the group is the step
    hbm, peak_kind = peaks()
    all_alg = sum(algorithmic_bytes(st, gg, nnz_before[i], nnz_after[i])
                  for i, gg in enumerate(st.groups))
    achieved = all_alg / (ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_r02.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("step")
        except Exception:
            traffic = None
    order, _ = st.step_plans()
    per_class = timed_serial_classes(st, 3, stream, HYPER)
    st.check()
    for g in order[:-1]:  # restore the concurrent caps
        q._native.check(q._native.lib.qftc_plan_set_ctas_per_sm(
            g.plan, int(os.environ.get("QFT_WIDE_CTAS", "0"))))

    # ---------------- e2e: the reference-facing call with HOST buffers ----------------
    e2e = e2e_host(st, q, args, stream) if not args.no_e2e else None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (device generator, bit-identical to oracle/synth.c)",
        "config": {"workload": "llama2-7b-shaped full model-state quantized Lion step "
                               "(configs[1]): 291 tensors, 6.74 G params, b=8, p=1% percentile "
                               "outliers, u8 gradient codes",
                   "params": params_local, "rows": rows_local, "bit_width": BIT_WIDTH,
                   "outlier_fraction": FRACTION, "nnz": st.nnz(), "lr": HYPER["lr"],
                   "l2": "inputs larger than L2 (34.8 GB moved per step vs 126 MB L2)",
                   "parallelism": "single"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "kernel": "qftc_plans_step: the width classes' launch groups (k_step_prep "
                               "+ rows_kernel, stable tier + step_kernel, general tier) forked "
                               "onto concurrent streams -- one launch group per step",
                     "algorithmic_bytes_per_launch": all_alg, "launch_ms": ms,
                     "peak_kind": peak_kind},
        "step_hbm_gbs": achieved,
        "step_frac": achieved / hbm,
        "stable_rows_frac": st_rows / max(1, st_rows + gen_rows),
        "tier_rows": {"stable": tiers[0], "gen": tiers[1], "general": tiers[2]},
        "per_class_serial_ms": {f"cols{gg.cols}": per_class[i] for i, gg in enumerate(st.groups)},
        "per_class_serial_frac": {
            f"cols{gg.cols}": algorithmic_bytes(st, gg, nnz_before[i], nnz_after[i]) /
            (per_class[i] * 1e-3) / 1e9 / hbm for i, gg in enumerate(st.groups)},
        "concurrency": {"wide_class_ctas_per_sm": int(os.environ.get("QFT_WIDE_CTAS", "0")),
                        "order": [f"cols{g.cols}" for g in order]},
        "gpu_launches": args.steps * sum(int(q._native.lib.qftc_plan_launches(gg.plan)) for gg in st.groups),
        "clocks": clocks,
        "setup_s": setup_s,
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_side:
        # the general tier: lr = 2.2e-4 puts rows on both sides of the stable-tier bound
        try:
            line["side_lr_2.2e-4"] = side_lr(st, args, stream, all_alg, hbm)
        except Exception as ex:  # a side measurement never voids the headline
            line["side_lr_2.2e-4"] = {"error": str(ex)[:300]}
    del st
    torch.cuda.empty_cache()
    if not args.no_side:
        try:
            line["side_bf16_grad"] = side_bf16(args, full, q, stream, hbm)
        except Exception as ex:
            line["side_bf16_grad"] = {"error": str(ex)[:300]}
        torch.cuda.empty_cache()
    if args.zero1:
        line["zero1_step"] = zero1_run(args, full, world, rank, q)
        torch.cuda.empty_cache()
        try:
            line["zero1_fused_step"] = zero1_fused_run(args, full, world, rank, q)
        except Exception as ex:  # a side measurement never voids the headline
            line["zero1_fused_step"] = {"error": str(ex)[:300]}
    if not args.no_cpu:
        try:
            cb = cpu_reference_run(steps=2, warmup=0)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind",
                                                       "sample", "cpu_model")}
        except Exception as ex:  # reported, never fatal for the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    print(json.dumps(line), flush=True)


def timed_region(st, steps, stream, hyper):
    """`steps` fused steps over the whole model: one concurrent launch group per step (every
    width class on its own stream, qftc_plans_step); ms per step from CUDA events on the
    launching stream (the classes are forked from and joined back into it)."""
    import torch
    import paper_2310_07147_b200 as q
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    h = q._native.hyper(hyper["lr"], hyper["beta1"], hyper["beta2"], hyper["weight_decay"])
    sh = C.c_void_p(stream.cuda_stream)
    ev0.record(stream)
    for _ in range(steps):
        flip = st.cur
        st.enqueue_step(flip, h, sh)
        st.cur = 1 - flip
        st.steps += 1
    ev1.record(stream)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / steps


def timed_serial_classes(st, steps, stream, hyper):
    """Per width class: the classes stepped one after the other on one stream, uncapped
    grids, CUDA events around each class's launch group (mean ms per class)."""
    import torch
    import paper_2310_07147_b200 as q
    N = q._native
    for g in st.groups:
        N.check(N.lib.qftc_plan_set_ctas_per_sm(g.plan, 0))
    st._plan_order = None
    h = N.hyper(hyper["lr"], hyper["beta1"], hyper["beta2"], hyper["weight_decay"])
    sh = C.c_void_p(stream.cuda_stream)
    gev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in st.groups] for _ in range(steps)]
    for k in range(steps):
        flip = st.cur
        for gi, g in enumerate(st.groups):
            gev[k][gi][0].record(stream)
            N.check(N.lib.qftc_plan_step(g.plan, flip, h, sh))
            gev[k][gi][1].record(stream)
        st.cur = 1 - flip
        st.steps += 1
    torch.cuda.synchronize()
    return [statistics.mean(gev[k][gi][0].elapsed_time(gev[k][gi][1]) for k in range(steps))
            for gi in range(len(st.groups))]


def side_lr(st, args, stream, alg_step, hbm):
    """The same 7B state stepped at lr = 2.2e-4 (rows whose sw is
    below ~2*lr leave the stable tier and run the general step kernel; their codes move,
    so CSR slots can overflow).  Every step is the checked engine step (synchronise,
    re-plan + re-run on overflow), timed with CUDA events around it."""
    import torch
    hy = dict(HYPER, lr=2.2e-4)
    for _ in range(args.warmup):
        st.step(**hy, check=True)
    rp0 = st.replans
    n = min(args.steps, 5)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(n)]
    for e0, e1 in ev:
        e0.record(stream)
        st.step(**hy, check=True)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev)
    t3 = st.tiers()
    return {"lr": hy["lr"], "ms_per_step": ms, "gparams_s": st.param_count / (ms * 1e-3) / 1e9,
            "stable_rows_frac": t3[0] / max(1, sum(t3)),
            "tier_rows": {"stable": t3[0], "gen": t3[1], "general": t3[2]},
            "replans_in_timed_steps": st.replans - rp0,
            "step_frac_approx": alg_step / (ms * 1e-3) / 1e9 / hbm,
            "timing": "checked engine step (host sync per step) between CUDA events"}


def side_bf16(args, full, q, stream, hbm):
    """The 7B step fed raw bf16 gradients (what a reduce-scatter delivers): k_grad_quant
    (quantize_state of g into the u8 GradientStack entry) + the rows kernel, per group."""
    import torch
    st = q.QftModelState(full, bit_width=BIT_WIDTH, grad_kind="bf16")
    st.init_from_weights(lambda i: q.synth(full[i], 1234 + i, 0.02, 0.005), FRACTION, "percentile")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    st.g_raw.normal_(0.0, 1e-3, generator=gen)
    for _ in range(args.warmup):
        st.step(**HYPER, check=True)
    nnz0 = st.nnz()
    ms = timed_region(st, min(args.steps, 5), stream, HYPER)
    st.check()
    a, b = st.tier_rows()
    P, R = st.param_count, st.row_count_total
    # 2 B bf16 read + 1 B code write + 8 B params per row (k_grad_quant), then the u8 step
    alg = 3 * P + 8 * R + 5 * P + 8 * (nnz0 + st.nnz()) + 48 * R
    out = {"ms_per_step": ms, "gparams_s": P / (ms * 1e-3) / 1e9, "grad": "bf16 raw",
           "algorithmic_bytes": alg, "frac_of_hbm": alg / (ms * 1e-3) / 1e9 / hbm,
           "stable_rows_frac": a / max(1, a + b), "kernels": st.kernel_names(),
           "launches_per_step": sum(int(q._native.lib.qftc_plan_launches(g.plan))
                                    for g in st.groups)}
    del st
    torch.cuda.empty_cache()
    return out


def run_multi_gpu(args, full, world, rank, local, q):
    """configs[2] at N > 1: the headline is the FULL ZeRO-1 step (reduce-scatter of the
    bf16 gradient + local update + all-gather of the quantized state), device time max over
    ranks; the update alone and the collectives are side fields."""
    import torch
    import torch.distributed as dist
    from paper_2310_07147_b200.shapes import count
    clk = ClockSampler(local)
    clk.start()
    z = zero1_run(args, full, world, rank, q)
    clocks = clk.stop()
    torch.cuda.empty_cache()
    try:
        zf = zero1_fused_run(args, full, world, rank, q)
    except Exception as ex:  # a side measurement never voids the headline
        zf = {"error": str(ex)[:300]}
    hbm, peak_kind = peaks()
    params = count(full)[0]
    ms = z["ms_per_step"]
    d = z["dominant"]
    achieved = d["algorithmic_bytes"] / (d["ms"] * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": params / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (device generator; bf16 gradients from torch.normal on device)",
        "config": {"workload": "llama2-7b-shaped ZeRO-1 quantized Lion step (configs[2]): "
                               "reduce-scatter bf16 grad + per-shard fused update + all-gather "
                               "of W codes / CSR slots / arenas",
                   "params": params, "bit_width": BIT_WIDTH, "outlier_fraction": FRACTION,
                   "lr": HYPER["lr"], "parallelism": f"zero1-rows{world}",
                   "l2": "inputs larger than L2"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": None,
                     "kernel": "rank-local update: every width class's k_grad_quant + "
                               "k_step_prep + rows_kernel + step_kernel, concurrent streams",
                     "algorithmic_bytes_per_launch": d["algorithmic_bytes"],
                     "launch_ms": d["ms"], "peak_kind": peak_kind},
        "zero1_step": z,
        "zero1_fused_step": zf,
        "update_only_gparams_s": z["update_gparams_s_all_ranks"],
        "gpu_launches": args.steps * z["gpu_launches_per_step"],
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def zero1_fused_run(args, full, world, rank, q):
    """§8(f) row 3: the ZeRO-1 step over peer memory (CUDA IPC mappings instead of NCCL):
    the reduce-scatter fused into the update's gradient quantizer (k_rs_grad_quant reads
    every rank's bf16 rows and quantizes their fp32 sum in one pass), then the push
    all-gather.  Device time between CUDA events around the whole step (its host barriers
    included), max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2310_07147_b200.zero1 import CudaShard, ShardLayout, Zero1QftLion
    own_group = not dist.is_initialized()
    if own_group:
        import socket
        s_ = socket.socket()
        s_.bind(("127.0.0.1", 0))
        port_no = s_.getsockname()[1]
        s_.close()
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_no}", rank=0,
                                world_size=1)
    try:
        layout = ShardLayout(full, world)
        local = CudaShard(layout, rank, bit_width=BIT_WIDTH, grad_dtype=torch.bfloat16)
        shard = layout.shard_shapes(rank)
        local.state.init_from_weights(
            lambda i: q.synth(shard[i], 4321 + 1000 * rank + i, 0.02, 0.005), FRACTION, "percentile")
        z = Zero1QftLion(full, local)
        z.enable_peer_memory()
        gen = torch.Generator(device="cuda")
        gen.manual_seed(99 + rank)
        z.grad_full.normal_(0.0, 1e-3 / world, generator=gen)
        stream = torch.cuda.current_stream()
        for _ in range(args.warmup):
            z.step_fused(**HYPER)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for e0, e1 in ev:
            e0.record(stream)
            z.step_fused(**HYPER)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev)
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        params = sum(r * c for r, c in full)
        z._close_peers()
        return {"ms_per_step": ms, "gparams_s": params / (ms * 1e-3) / 1e9, "world": world,
                "what": "fused reduce-scatter + quantize_state over peer memory (k_rs_grad_quant), "
                        "rows kernels, push all-gather; host barriers included",
                "kernels": local.state.kernel_names()}
    finally:
        if own_group:
            dist.destroy_process_group()


def zero1_run(args, full, world, rank, q):
    """configs[2]: the full ZeRO-1 step on this rank -- reduce-scatter of the bf16
    gradient (shard-major layout), the local update of the rank's rows (k_grad_quant:
    quantize_state of the summed bf16 gradient into the u8 GradientStack entry, then the
    rows kernel), all-gather of the updated W codes, CSR slot starts/counts and arenas.
    Device time per phase (CUDA events on the launching stream), max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2310_07147_b200.zero1 import CudaShard, ShardLayout, Zero1QftLion
    own_group = not dist.is_initialized()
    if own_group:  # single-process check of the path (bench.py --zero1 at N=1)
        import socket
        s_ = socket.socket()
        s_.bind(("127.0.0.1", 0))
        port_no = s_.getsockname()[1]
        s_.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port_no}", rank=0,
                                world_size=1)
    try:
        layout = ShardLayout(full, world)
        local = CudaShard(layout, rank, bit_width=BIT_WIDTH, grad_dtype=torch.bfloat16)
        shard = layout.shard_shapes(rank)
        local.state.init_from_weights(
            lambda i: q.synth(shard[i], 4321 + 1000 * rank + i, 0.02, 0.005), FRACTION, "percentile")
        z = Zero1QftLion(full, local)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(99 + rank)
        z.grad_full.normal_(0.0, 1e-3 / world, generator=gen)
        g0 = z.grad_full.clone()
        st = local.state
        stream = torch.cuda.current_stream()
        for _ in range(args.warmup):
            z.grad_full.copy_(g0)
            z.step(**HYPER)
            st.check()
        dist.barrier()
        torch.cuda.synchronize()
        nnz_before = [st.group_nnz(g) for g in st.groups]
        E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        ev = [(E(), E(), E(), E(), E()) for _ in range(args.steps)]
        h = _hyper_c()
        for e0, e1, e15, e2, e3 in ev:
            z.grad_full.copy_(g0)       # a fresh gradient each step (outside the event pairs)
            e0.record(stream)
            z.reduce_scatter_grads()
            e1.record(stream)
            flip = st.cur
            st.enqueue_step(flip, h, C.c_void_p(stream.cuda_stream))
            e15.record(stream)
            st.cur = 1 - flip
            st.steps += 1
            z.check_local()             # all-reduced overflow flag (re-plans + re-runs)
            e2.record(stream)
            z.all_gather_state()
            e3.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        st.check()
        nnz_after = [st.group_nnz(g) for g in st.groups]
        mean = lambda a, b: statistics.mean(x.elapsed_time(y) for x, y in zip(a, b))  # noqa: E731
        ms = mean([e[0] for e in ev], [e[4] for e in ev])
        rs_ms = mean([e[0] for e in ev], [e[1] for e in ev])
        upd_ms = mean([e[1] for e in ev], [e[3] for e in ev])
        ag_ms = mean([e[3] for e in ev], [e[4] for e in ev])
        kern_ms = mean([e[1] for e in ev], [e[2] for e in ev])
        t = torch.tensor([ms, rs_ms, upd_ms, ag_ms, kern_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, rs_ms, upd_ms, ag_ms, kern_ms = (float(x) for x in t.tolist())
        params = sum(r * c for r, c in full)
        shard_params = st.param_count
        f = (world - 1) / world
        rs_bytes = f * 2 * layout.pad * world
        ag_bytes = f * z.gather_bytes_per_rank() * world   # packed: only used CSR entries
        # the update's launch group: k_grad_quant (2 B bf16 read + 1 B code write per param,
        # 8 B params per row) + the step on the u8 entry (5 B per param,
        # 8 B per CSR entry in and out, 48 B per row), every width class concurrently
        alg = sum(3 * sum(st.shapes[i][0] * st.shapes[i][1] for i in g.members) + 8 * g.rows +
                  algorithmic_bytes(st, g, nnz_before[gi], nnz_after[gi])
                  for gi, g in enumerate(st.groups))
        st_, gen_ = st.tier_rows()
        return {"ms_per_step": ms, "gparams_s": params / (ms * 1e-3) / 1e9,
                "what": "reduce_scatter(bf16 grad) + local update of the row shard "
                        "(k_grad_quant -> rows kernel) + all_gather(W codes, CSR slots, arenas)",
                "grad_dtype": "bf16", "world": world, "shard_params": shard_params,
                "rs_ms": rs_ms, "update_ms": upd_ms, "ag_ms": ag_ms,
                "update_gparams_s_per_rank": shard_params / (upd_ms * 1e-3) / 1e9,
                "update_gparams_s_all_ranks": params / (upd_ms * 1e-3) / 1e9,
                "dominant": {"what": "the local update's concurrent launch group (all width "
                                     "classes)", "ms": kern_ms, "algorithmic_bytes": alg},
                "stable_rows_frac": st_ / max(1, st_ + gen_),
                "rs_bytes_per_rank": rs_bytes, "ag_bytes_per_rank": ag_bytes,
                "nvlink_gbs_per_rank": (rs_bytes + ag_bytes) / ((rs_ms + ag_ms) * 1e-3) / 1e9,
                "nccl_version": ".".join(str(v) for v in torch.cuda.nccl.version()),
                "gpu_launches_per_step": sum(int(q._native.lib.qftc_plan_launches(gg.plan))
                                             for gg in st.groups)}
    finally:
        if own_group:
            dist.destroy_process_group()


def e2e_host(st, q, args, stream):
    """End-to-end through the reference-facing call with HOST buffers: every step
    uploads the whole host-resident state the reference API passes by reference
    (Model weights: codes, CSR; LionState momentum) plus the GradientStack entry,
    runs the fused step, and reads the updated state back -- all copies from/to
    pinned host memory inside the timed region.  The model is cut into ~256 M-param
    chunks (one plan each) and three streams overlap H2D of chunk i+1, the fused
    step on chunk i and D2H of chunk i-1 (PCIe is full duplex)."""
    import torch

    N = q._native
    chunks = st.make_chunk_plans(256 << 20)
    k0 = st.cur
    if not torch.equal(st.row_start[0], st.row_start[1]):
        st._mirror_all()  # one host copy needs one slot layout for both sets
    ranges = [st.chunk_ranges(ch, k0) for ch in chunks]

    def dev_state(k):
        d = {"w_codes": st.w_codes[k], "m_codes": st.m_codes[k], "m_scale": st.m_scale[k],
             "m_zp": st.m_zp[k], "row_start": st.row_start[k], "row_count": st.row_count[k]}
        for gi, g in enumerate(st.groups):
            d[f"col{gi}"], d[f"val{gi}"] = g.col[k], g.val[k]
        return d

    kind = {"w_codes": "code", "m_codes": "code", "m_scale": "row", "m_zp": "row",
            "row_start": "rs", "row_count": "row"}
    grads = {"g_codes": (st.g_codes, "code"), "g_scale": (st.g_scale, "row"),
             "g_zp": (st.g_zp, "row")}
    host = {n: torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
            for n, t in dev_state(k0).items()}
    for n, t in dev_state(k0).items():
        host[n].copy_(t)
    for n, (t, _) in grads.items():
        host[n] = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
        host[n].copy_(t)

    def rng(n, ci):
        r = ranges[ci]
        if n.startswith("col") or n.startswith("val"):
            return r["arena"] if int(n[3:]) == st.groups.index(chunks[ci]["group"]) else None
        return r[kind[n] if n in kind else grads[n][1]]

    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()
    in_done = [ev() for _ in chunks]
    cmp_done = [ev() for _ in chunks]
    out_done = [ev() for _ in chunks]
    h = N.hyper(HYPER["lr"], HYPER["beta1"], HYPER["beta2"], HYPER["weight_decay"])
    steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    s_out.wait_event(e0)
    s_cmp.wait_event(e0)
    h2d = d2h = 0
    for _ in range(steps):
        c_in = st.cur
        src, dst = dev_state(c_in), dev_state(1 - c_in)
        h2d = d2h = 0
        for ci, ch in enumerate(chunks):
            with torch.cuda.stream(s_in):
                s_in.wait_event(out_done[ci])
                for n, t in list(src.items()) + [(n, g) for n, (g, _) in grads.items()]:
                    r = rng(n, ci)
                    if r is None or r[1] <= r[0]:
                        continue
                    t[r[0]:r[1]].copy_(host[n][r[0]:r[1]], non_blocking=True)
                    h2d += (r[1] - r[0]) * t.element_size()
                in_done[ci].record(s_in)
            s_cmp.wait_event(in_done[ci])
            st.step_chunk(ch, c_in, h, C.c_void_p(s_cmp.cuda_stream))
            cmp_done[ci].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(cmp_done[ci])
                for n, t in dst.items():
                    r = rng(n, ci)
                    if r is None or r[1] <= r[0]:
                        continue
                    host[n][r[0]:r[1]].copy_(t[r[0]:r[1]], non_blocking=True)
                    d2h += (r[1] - r[0]) * t.element_size()
                out_done[ci].record(s_out)
        st.cur = 1 - c_in
        st.steps += 1
    e1.record(s_out)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    st.check()
    return {"value": st.param_count / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "chunks": len(chunks),
            "what": "full host-resident state + gradient in, updated state out (pinned), "
                    "chunked 3-stream H2D/step/D2H overlap"}


def timed_steps(st, steps, stream):
    """device time per launch group and per step for `steps` fused steps"""
    import torch
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in st.groups] for _ in range(steps)]
    h = None
    for k in range(steps):
        flip = st.cur
        for gi, g in enumerate(st.groups):
            ev[k][gi][0].record(stream)
            st.step_chunk({"plan": g.plan}, flip, _hyper_c(), C.c_void_p(stream.cuda_stream))
            ev[k][gi][1].record(stream)
        st.cur = 1 - flip
    torch.cuda.synchronize()
    st.check()
    per = [statistics.mean(ev[k][gi][0].elapsed_time(ev[k][gi][1]) for k in range(steps))
           for gi in range(len(st.groups))]
    return per


def _hyper_c():
    import paper_2310_07147_b200 as q
    return q._native.hyper(HYPER["lr"], HYPER["beta1"], HYPER["beta2"], HYPER["weight_decay"])


def run_sweep(args):
    """configs[4]: weight bit width x outlier fraction on LLaMA-2-7B's 32 down-proj
    tensors (4096 x 11008, 1.44 G params: out of L2), bytes/param vs roofline."""
    import torch
    import paper_2310_07147_b200 as q
    global BIT_WIDTH, FRACTION
    hbm, _ = peaks()
    shapes = [(4096, 11008)] * 32
    stream = torch.cuda.current_stream()
    rows = []
    for bw in (3, 4, 8):
        for frac in (0.0005, 0.001, 0.0045, 0.01):
            BIT_WIDTH, FRACTION = bw, frac
            st = build_state(shapes, q, 777)
            for _ in range(args.warmup):
                st.step(**HYPER, check=True)
            nnz0 = st.nnz()
            per = timed_steps(st, args.steps, stream)
            nnz1 = st.nnz()
            params = st.param_count
            alg = 5 * params + 8 * (nnz0 + nnz1) + 48 * st.row_count_total
            ms = sum(per)
            rows.append({"bit_width": bw, "outlier_fraction": frac, "ms": ms,
                         "gparams_s": params / (ms * 1e-3) / 1e9,
                         "bytes_per_param": alg / params, "achieved_gbs": alg / (ms * 1e-3) / 1e9,
                         "frac_of_hbm": alg / (ms * 1e-3) / 1e9 / hbm, "nnz": nnz1})
            del st
            torch.cuda.empty_cache()
    print(json.dumps({"sweep": "llama2-7b down_proj x32 (4096x11008), reference u8 layout",
                      "peak_gbs": hbm, "rows": rows}), flush=True)


def run_13b_dequant(args):
    """configs[3] per rank, on one GPU: rank 0 of 8's row shard of LLaMA-2-13B stepped with
    the bf16 gradient a reduce-scatter delivers (k_grad_quant -> rows kernels, width classes
    concurrent), then the next forward's bf16 weights of the WHOLE model expanded in ONE
    launch straight from the all-gathered, shard-major buffers (Zero1QftLion.expand_plan).
    The 8 ranks' gathered content is rank 0's shard for ranks 0-6 and rank 7's (which also
    holds the 1-row norms) -- the same layout and byte counts as a real all-gather; the
    collectives themselves need 8 GPUs."""
    import torch
    import paper_2310_07147_b200 as q
    from paper_2310_07147_b200.shapes import llama2_13b
    from paper_2310_07147_b200.zero1 import CudaShard, ShardLayout, Zero1QftLion
    hbm, _ = peaks()
    full = llama2_13b()
    world = 8
    L = ShardLayout(full, world)
    stream = torch.cuda.current_stream()
    shards = {}
    for k in (0, world - 1):
        sh = CudaShard(L, k, bit_width=BIT_WIDTH, grad_dtype=torch.bfloat16)
        ss = L.shard_shapes(k)
        sh.state.init_from_weights(lambda i, ss=ss, k=k: q.synth(ss[i], 1313 + 1000 * k + i, 0.02, 0.005),
                                   FRACTION, "percentile")
        gen = torch.Generator(device="cuda")
        gen.manual_seed(5 + k)
        sh.state.g_raw.normal_(0.0, 1e-3, generator=gen)
        shards[k] = sh
    st = shards[0].state
    for _ in range(args.warmup):
        st.step(**HYPER, check=True)
    nnz0 = st.nnz()
    step_ms = timed_region(st, args.steps, stream, HYPER)
    st.check()
    P, R = st.param_count, st.row_count_total
    step_alg = 3 * P + 8 * R + 5 * P + 8 * (nnz0 + st.nnz()) + 48 * R
    # the all-gathered buffers (all_gather_into_tensor layout: rank-major, uniform sizes)
    cap = max(s.arena_capacity() for s in shards.values())
    for s in shards.values():
        s.ensure_arena_capacity(cap)
    src = [shards[0]] * (world - 1) + [shards[world - 1]]
    z = Zero1QftLion.__new__(Zero1QftLion)
    z.layout, z.world, z.cap, z.local = L, world, cap, shards[0]
    z.codes_full = torch.cat([s.codes_shard(L.pad) for s in src])
    z.rowstart_full = torch.cat([s.rowstart_shard(L.rp_pad) for s in src])
    z.count_full = torch.cat([s.count_shard(L.rpad) for s in src])
    z.wscale_full = torch.cat([s.wscale_shard(L.rpad) for s in src])
    z.wzp_full = torch.cat([s.wzp_shard(L.rpad) for s in src])
    z.col_full, z.val_full = {}, {}
    for c in L.widths:
        cols, vals = zip(*[s.arena(c, cap) for s in src])
        z.col_full[c], z.val_full[c] = torch.cat(cols), torch.cat(vals)
    outs = [torch.empty((r, c), dtype=torch.bfloat16, device="cuda") for r, c in full]
    plan = z.expand_plan(outs)
    for _ in range(2):
        plan.run()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    for e0, e1 in ev:
        e0.record(stream)
        plan.run()
        e1.record(stream)
    torch.cuda.synchronize()
    dq_ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in ev)
    n_el = sum(r * c for r, c in full)
    cnt = z.count_full.view(world, L.rpad)
    nnz = int(sum(int(cnt[k, :L.rows[k]].sum().item()) for k in range(world)))
    rows_all = sum(r for r, _ in full)
    # 1 B code read + 2 B bf16 written per param, 8 B per CSR entry read (+2 B scattered
    # bf16 write), 16 B per row (scale, zp, slot start, count)
    dq_bytes = 3 * n_el + 10 * nnz + 16 * rows_all
    print(json.dumps({
        "config": "llama2-13b per rank of 8 (configs[3]): row-shard step fed bf16 reduce-scatter "
                  "gradients + the whole model's bf16 weights expanded from the all-gathered "
                  "shard-major buffers", "shard_params": P,
        "step_ms": step_ms, "step_gparams_s": P / (step_ms * 1e-3) / 1e9,
        "step_frac_of_hbm": step_alg / (step_ms * 1e-3) / 1e9 / hbm,
        "step_kernels": st.kernel_names(),
        "dequant_params": n_el, "dequant_nnz": nnz, "dequant_ms": dq_ms,
        "dequant_launches": 1, "dequant_table_entries": plan.n,
        "dequant_gparams_s": n_el / (dq_ms * 1e-3) / 1e9,
        "dequant_gbs": dq_bytes / (dq_ms * 1e-3) / 1e9,
        "dequant_frac_of_hbm": dq_bytes / (dq_ms * 1e-3) / 1e9 / hbm,
        "per_rank_compute_ms": step_ms + dq_ms, "peak_gbs": hbm}), flush=True)


def run_gemm(args):
    """the forward GEMM of a LLaMA-2-7B layer's projections with the
    weight dequantization fused into its operand producer (QftModelState.linear ->
    qftc_dequant_gemm, tcgen05 + TMA), against the materialised path (bf16 expansion of the
    weight, qftc_expand, + cuBLAS torch.matmul) and cuBLAS alone on pre-expanded weights."""
    import torch
    import paper_2310_07147_b200 as q
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak_tf = float(pk.get("bf16_tflops", 2250.0))
    tokens = 4096  # a micro-batch of 8 x 512 tokens
    stream = torch.cuda.current_stream()
    out = []
    for name, (r, c) in (("q/k/v/o", (4096, 4096)), ("gate/up", (11008, 4096)),
                         ("down", (4096, 11008))):
        st = q.QftModelState([(r, c)], bit_width=BIT_WIDTH)
        st.init_from_weights(lambda i: q.synth((r, c), 4242, 0.02, 0.005), FRACTION, "percentile")
        x = (torch.randn(tokens, c, device="cuda") * 0.5).to(torch.bfloat16)
        wb = torch.empty((r, c), dtype=torch.bfloat16, device="cuda")
        y = torch.empty((tokens, r), dtype=torch.bfloat16, device="cuda")
        plan = st.expand_plan([wb])

        def timeit(fn, n=max(args.steps, 10)):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(n):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n

        # the CSR slot index is a function of the weight: built once per weight version
        # (csr_index, timed on its own) and reused by the micro-batches' GEMMs; the per-call
        # form (index rebuilt inside every call) is reported beside it
        idx = st.csr_index(0)
        index_ms = timeit(lambda: st.csr_index(0))
        fused = timeit(lambda: st.linear(0, x, out=y, index=idx))
        fused_rebuild = timeit(lambda: st.linear(0, x, out=y))
        dy = (torch.randn(tokens, r, device="cuda") * 0.5).to(torch.bfloat16)
        dx = torch.empty((tokens, c), dtype=torch.bfloat16, device="cuda")
        fused_t = timeit(lambda: st.linear_backward(0, dy, out=dx, index=idx))
        fused_t_rebuild = timeit(lambda: st.linear_backward(0, dy, out=dx))
        mat = timeit(lambda: (plan.run(), torch.matmul(x, wb.t(), out=y)))
        plan.run()
        cublas = timeit(lambda: torch.matmul(x, wb.t(), out=y))
        mat_t = timeit(lambda: (plan.run(), torch.matmul(dy, wb, out=dx)))
        cublas_t = timeit(lambda: torch.matmul(dy, wb, out=dx))
        flops = 2.0 * tokens * r * c
        out.append({"proj": name, "M": tokens, "N": r, "K": c,
                    "fused_ms": fused, "fused_tflops": flops / fused / 1e9,
                    "csr_index_ms": index_ms,
                    "fused_with_index_rebuild_ms": fused_rebuild,
                    "backward_dx_fused_with_index_rebuild_ms": fused_t_rebuild,
                    "fused_frac_of_bf16_peak": flops / fused / 1e9 / peak_tf,
                    "expand_plus_cublas_ms": mat, "cublas_only_ms": cublas,
                    "cublas_tflops": flops / cublas / 1e9,
                    "backward_dx_fused_ms": fused_t,
                    "backward_dx_fused_tflops": flops / fused_t / 1e9,
                    "backward_dx_expand_plus_cublas_ms": mat_t,
                    "backward_dx_cublas_only_ms": cublas_t,
                    "weight_bytes_read_fused": r * c + 10 * st.nnz() + 16 * r,
                    "weight_bytes_materialised": 3 * r * c + 2 * r * c})
        del st, x, wb, y, plan, dy, dx
        torch.cuda.empty_cache()
    print(json.dumps({"gemm": "y = x . W^T, W dense-and-sparse (b=8, p=1%), x/y bf16, "
                              "fused dequant (tcgen05) vs expand + cuBLAS",
                      "bf16_peak_tflops": peak_tf, "rows": out}), flush=True)


def run_wgrad(args):
    """the backward's weight gradient G = dy^T . x of a LLaMA-2-7B
    layer's projections with the sink's quantize_state fused into the GEMM epilogue
    (QftModelState.sink_wgrad -> qftc_wgrad_quant, tcgen05 + TMA, MN-major operands; the
    fp32 gradient never reaches HBM), against the materialised path: cuBLAS bf16 GEMM with
    fp32 output (torch.mm out_dtype=float32) + the quantize_state row kernel, and cuBLAS
    alone.  Both the push (first micro-batch) and the accumulate form are timed."""
    import torch
    import paper_2310_07147_b200 as q
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak_tf = float(pk.get("bf16_tflops", 2250.0))
    tokens = 4096  # a micro-batch of 8 x 512 tokens
    stream = torch.cuda.current_stream()
    out = []
    for name, (r, c) in (("q/k/v/o", (4096, 4096)), ("gate/up", (11008, 4096)),
                         ("down", (4096, 11008))):
        st = q.QftModelState([(r, c)], bit_width=BIT_WIDTH)
        st.init_from_weights(lambda i: q.synth((r, c), 4242, 0.02, 0.005), FRACTION, "percentile")
        dy = (torch.randn(tokens, r, device="cuda") * 1e-2).to(torch.bfloat16)
        x = torch.randn(tokens, c, device="cuda").to(torch.bfloat16)
        g = torch.empty((r, c), dtype=torch.float32, device="cuda")
        codes, s, z = st.grad_views(0)

        def timeit(fn, n=max(args.steps, 10)):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(n):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n

        fused = timeit(lambda: st.sink_wgrad(0, dy, x))
        fused_acc = timeit(lambda: st.sink_wgrad(0, dy, x, accumulate=True))

        from paper_2310_07147_b200 import _native as NN
        from paper_2310_07147_b200.quantize import _p, _stream

        def materialised():  # no host synchronisation (check = 0), like the fused call
            torch.mm(dy.t(), x, out_dtype=torch.float32, out=g)
            NN.check(NN.lib.qftc_quantize_state(_p(g), r, c, BIT_WIDTH, _p(codes), _p(s), _p(z),
                                                0, _stream()))

        mat = timeit(materialised)
        cublas = timeit(lambda: torch.mm(dy.t(), x, out_dtype=torch.float32, out=g))
        flops = 2.0 * tokens * r * c
        out.append({"proj": name, "out": r, "in": c, "tokens": tokens,
                    "fused_ms": fused, "fused_tflops": flops / fused / 1e9,
                    "fused_frac_of_bf16_peak": flops / fused / 1e9 / peak_tf,
                    "fused_accumulate_ms": fused_acc,
                    "cublas_f32_plus_quantize_state_ms": mat,
                    "cublas_f32_only_ms": cublas, "cublas_tflops": flops / cublas / 1e9,
                    "gradient_bytes_written_fused": r * c + 8 * r,
                    "gradient_bytes_materialised": 4 * r * c + 4 * r * c + r * c + 8 * r})
        del st, dy, x, g
        torch.cuda.empty_cache()
    print(json.dumps({"wgrad": "G = dy^T . x, quantize_state(G) (b=8) in the GEMM epilogue "
                               "(tcgen05) vs cuBLAS f32-output GEMM + quantize_state kernel",
                      "bf16_peak_tflops": peak_tf, "rows": out}), flush=True)


def run_ckpt(args):
    """QFTC v1 checkpoint of the 7B state: the GPU CRC-32
    over every array of the file in file order (HBM-resident, ~13.8 GB), zlib.crc32 on
    one host core over a 256 MB sample for scale, and save + load of one LLaMA-2-7B
    decoder layer (9 tensors, 202 M params) through paper_2310_07147_b200.checkpoint."""
    import tempfile
    import time
    import zlib

    import torch
    import paper_2310_07147_b200 as q
    from paper_2310_07147_b200.checkpoint import _crc_device, load_checkpoint, save_checkpoint
    from paper_2310_07147_b200.shapes import llama2_7b
    hbm, _ = peaks()
    shapes = llama2_7b()
    st = build_state(shapes, q, 1234)
    segs = []
    for i in range(st.n):
        rp, col, val = st.strict_csr(i)
        segs += [st._rows(st.t_min, i), st._rows(st.t_max, i), st._rows(st.w_scale, i),
                 st._rows(st.w_zp, i), st._sl(st.w_codes[st.cur], i), rp, col, val,
                 st._rows(st.m_scale[st.cur], i), st._rows(st.m_zp[st.cur], i),
                 st._sl(st.m_codes[st.cur], i)]
    nbytes = sum(t.numel() * t.element_size() for t in segs)
    for _ in range(args.warmup):
        _crc_device(segs)
    ts, dev_ms = [], []
    stream = torch.cuda.current_stream()
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        _crc_device(segs)  # synchronises (chunk fold on the host)
        e1.record(stream)
        ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        dev_ms.append(e0.elapsed_time(e1))
    crc_s = statistics.median(ts)
    sample = torch.randint(0, 256, (256 << 20,), dtype=torch.uint8).numpy().tobytes()
    t0 = time.perf_counter()
    zlib.crc32(sample)
    zlib_gbs = len(sample) / (time.perf_counter() - t0) / 1e9
    del st, segs
    torch.cuda.empty_cache()
    one = shapes[1:10]  # one decoder layer: 2 norms + 7 matrices
    st1 = build_state(one, q, 77)
    with tempfile.TemporaryDirectory() as d:
        path = d + "/layer.qftc"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        save_checkpoint(st1, path)
        save_s = time.perf_counter() - t0
        size = os.path.getsize(path)
        t0 = time.perf_counter()
        st2, _ = load_checkpoint(path)
        torch.cuda.synchronize()
        load_s = time.perf_counter() - t0
    print(json.dumps({"config": "QFTC v1 checkpoint, llama2-7b state", "bytes": nbytes,
                      "gpu_crc_ms": crc_s * 1e3, "gpu_crc_gbs": nbytes / crc_s / 1e9,
                      "gpu_crc_frac_of_hbm": nbytes / crc_s / 1e9 / hbm,
                      "gpu_crc_device_ms": statistics.median(dev_ms),
                      "host_zlib_crc_gbs_1core": zlib_gbs,
                      "save_load_sample": f"{len(one)} tensors, {st1.param_count} params, "
                                          f"{size} bytes", "save_s": save_s, "load_s": load_s,
                      "timing": "wall clock around synchronous calls (median of steps)"}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--mode", default="step", choices=["step", "sweep", "13b", "ckpt", "gemm", "wgrad"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-side", action="store_true",
                    help="skip the lr=2.2e-4 and bf16-gradient side measurements")
    ap.add_argument("--zero1", action="store_true",
                    help="also time the full ZeRO-1 step (RS + step + AG) at N=1")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        s_ = socket.socket()
        s_.bind(("127.0.0.1", 0))
        port_no = s_.getsockname()[1]
        s_.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port_no}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.warmup < 3 and args.impl == "own":
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.mode == "sweep":
        run_sweep(args)
    elif args.mode == "13b":
        run_13b_dequant(args)
    elif args.mode == "ckpt":
        run_ckpt(args)
    elif args.mode == "gemm":
        run_gemm(args)
    elif args.mode == "wgrad":
        run_wgrad(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
