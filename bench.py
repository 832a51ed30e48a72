"""Benchmark: consistent MP-layer stack (forward + backward) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU)

Workload (BASELINE.json configs[2] at N=1): 32^3-element GLL box at P=5
(4,173,281 nodes, 24,884,160 directed edges), hidden 64, 5 hidden blocks per
MLP, 4 MP layers, exchange mode na2a. N>1 runs the weak-scaling series of
configs[4] (~4.2M nodes per GPU: E = 40/50/64 at N = 2/4/8, balanced block
partition), one GPU per rank, NCCL halo exchange over NVLink.
--scaling strong keeps one mesh at every N (configs[3]; E = 40 by default,
--elements 64 for the 33M-node box from N = 4); --mode a2a|none switches the
halo exchange (configs[4]'s comparison; none = the inconsistent baseline).

metric: MP-layer graph nodes per second, fwd+bwd
        = (unique global nodes) x (MP layers) / (time of one MP-stack fwd+bwd step)
value: device-resident inputs (synthetic, keyed by global id), CUDA events on
       the engine stream, max over ranks.
e2e:   same metric through the public C-ABI with fp64 host buffers in the
       reference layout (x0, e0, dx_M H2D; parameter gradients D2H) per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

LOADING = 4_173_281  # configs[2] nodes per GPU
P_ORDER, HIDDEN, M_LAYERS, K_HIDDEN = 5, 64, 4, 5
METRIC = "MP-layer graph nodes/sec (fwd+bwd)"
UNIT = "layer-nodes/s"


def choose_elements_for_loading(ranks: int, loading: int, p: int) -> int:
    """harness.cpp:271-296 (mesh sizing rule of the reference weak-scaling harness)."""
    from paper_2410_01657_b200 import PartitionError, balanced_factors
    best, best_err = -1, 0.0
    for e in range(1, 97):
        feasible = e % ranks == 0 and ranks <= e
        if not feasible:
            try:
                balanced_factors(ranks, e)
                feasible = True
            except PartitionError:
                feasible = False
        if not feasible:
            continue
        per_rank = (e * p + 1) ** 3 / ranks
        err = abs(per_rank - loading)
        if best < 0 or err < best_err:
            best, best_err = e, err
    return best


STRONG_E = 40  # strong-scaling default: 201^3 = 8.1M nodes, fits one GPU (configs[3]'s E = 64 fits from N = 4)


def workload(n_gpus: int, scaling: str = "weak", mode: str = "na2a"):
    """weak: configs[2] at N = 1, configs[4]'s ~4.2M nodes per GPU at N > 1.
    strong: one fixed mesh at every N (configs[3]; E = STRONG_E unless --elements)."""
    if scaling == "strong":
        E = STRONG_E
    else:
        E = 32 if n_gpus == 1 else choose_elements_for_loading(n_gpus, LOADING, P_ORDER)
    return {"E": E, "p": P_ORDER, "H": HIDDEN, "M": M_LAYERS, "k": K_HIDDEN, "mode": mode,
            "scaling": scaling, "unique_nodes": (E * P_ORDER + 1) ** 3}


def edge_flops(H, k):
    return 2 * H * H * (4 + k)


def node_flops(H, k):
    return 2 * H * H * (3 + k)


def edge_flops_fact(H, k):
    """Per edge in the factorised edge kernels (edge_factorized = 1): the input
    linear's x_src / x_dst blocks run at node level (edge_proj, node-level
    adjoint), the edge kernels multiply e W0_e, the k hidden and the output linear."""
    return 2 * H * H * (2 + k)


# --------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# --------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            f = [t.strip() for t in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        if not sm:
            return None
        under_load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(under_load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
# CPU reference timing (oracle/_ref = the reference compiled in place; else the
# C restatement). Test infrastructure: only this leg executes oracle/.
# --------------------------------------------------------------------------
REF_E = 6  # reference-arm sample: 6^3-element P=5 box (29,791 nodes), the full configs[2] layer stack


def cpu_reference_sample(steps: int = 1, E: int = REF_E):
    """The reference's CPU MP stack (fwd + bwd of all M layers, fp64, OpenMP
    over every host thread) on a bounded sample of configs[2]: the same layer
    shapes (H, k, M, mode) on an E^3-element P=5 box. configs[2] itself (32^3)
    does not fit a host's RAM in fp64. Imports only oracle/
    (oracle/_ref = the reference compiled in place; else the C restatement):
    nothing from the product package runs on this leg."""
    import oracle as O
    H, M, k = HIDDEN, M_LAYERS, K_HIDDEN
    rng = np.random.default_rng(0)
    nodes = (E * P_ORDER + 1) ** 3
    cores = os.cpu_count() or 1
    times = []
    if O.ref_available():
        kind = "reference"
        g = O.RefGraph(E, P_ORDER, 1, "verify", features=False)
        rg = g.ranks[0]
        rows, ne = rg.num_local + rg.num_halo, rg.num_edges
        mp = rng.uniform(-0.05, 0.05, O.ref_lib().ref_mp_param_count(H, M, k))
        x0 = [rng.uniform(-1, 1, (rows, H))]
        e0 = [rng.uniform(-1, 1, (ne, H))]
        dx = [rng.uniform(-1e-2, 1e-2, (rows, H))]
        for _ in range(steps):
            run = O.ref_mp_run(g, H, M, k, "na2a", mp, x0, e0, dx)
            f_ms, b_ms = run.times_ms()  # the reference's own timers around run_mp_stack
            times.append((f_ms + b_ms) / 1e3)
            del run
        api = "gnn_forward + gnn_backward layer loops (oracle/_ref: the reference compiled in place)"
    else:  # the C restatement alone has no mesh builder; the reference build ships with the repo
        raise RuntimeError("oracle/_ref/libhgnn_ref.so not built (python paper_2410_01657_b200/build.py --oracle)")
    t = statistics.median(times)
    return {"value": nodes * M / t, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{M} MP layers fwd+bwd (fp64, OpenMP over {cores} host threads), {E}^3-element box at "
                      f"P={P_ORDER} ({nodes} nodes, {ne} directed edges), H={H}, k={k}, mode=na2a, R=1: the "
                      f"configs[2] layer stack on a smaller box; median of {len(times)} run(s), {t:.2f} s each",
            "seconds": t, "E": E, "nodes": nodes, "api": api}


def run_reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    n = a.gpus
    if rank != 0:
        return
    for _ in range(min(a.warmup, 1)):
        cpu_reference_sample(1, a.ref_elements)
    res = cpu_reference_sample(max(1, a.steps), a.ref_elements)
    wl = {"E": res["E"], "p": P_ORDER, "H": HIDDEN, "M": M_LAYERS, "k": K_HIDDEN, "mode": "na2a",
          "scaling": "weak", "unique_nodes": res["nodes"]}
    cfg = config_dict(wl, 1)
    cfg["workload"] += (" -- the reference CPU path (fp64) on a bounded sample of configs[2]: same layer shapes, "
                        f"{res['E']}^3 instead of 32^3 elements (32^3 needs > 62 GB host RAM in fp64)")
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": n,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": res["seconds"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (uniform random inputs "
            "and MP weights)", "config": cfg, "api": res["api"],
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(wl, n):
    return {"workload": f"consistent MP stack fwd+bwd, {wl['E']}^3-element GLL box P={wl['p']} "
                        f"({wl['unique_nodes']} nodes), H={wl['H']}, k={wl['k']}, M={wl['M']}, mode={wl['mode']}",
            "elements_per_axis": wl["E"], "poly_order": wl["p"], "hidden": wl["H"], "mlp_hidden_layers": wl["k"],
            "mp_layers": wl["M"], "mode": wl["mode"], "unique_nodes": wl["unique_nodes"],
            "partition": "single rank" if n == 1 else "balanced block (verify_partition, harness.cpp:42-45)",
            "parallelism": f"domain decomposition x{n}", "l2": "inputs larger than L2 (no flush needed)"}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-train-step", action="store_true")
    ap.add_argument("--ref-elements", type=int, default=REF_E)
    ap.add_argument("--elements", type=int, default=0, help="override E (debug)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no e2e / baseline / clocks")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: ~4.2M nodes per GPU (configs[4]); strong: one fixed mesh at every N (configs[3])")
    ap.add_argument("--mode", default="na2a", choices=["na2a", "a2a", "none"],
                    help="halo exchange mode (configs[4] compares all three; none = the inconsistent baseline)")
    ap.add_argument("--halo-sm-reserve", type=int, default=-1, help="SMs left to the exchange (-1: engine default)")
    ap.add_argument("--fact", type=int, default=-1, choices=[-1, 0, 1],
                    help="edge_factorized option (-1: engine default)")
    ap.add_argument("--opt", action="append", default=[], metavar="KEY=VALUE",
                    help="extra engine option (hgnn_set_option), e.g. tma_gather=0 (A/B runs)")
    ap.add_argument("--halo-overlap", type=int, default=1, choices=[0, 1],
                    help="1: forward exchange on a side stream, overlapped with the interior edges (N > 1)")
    a = ap.parse_args()
    if a.impl == "reference":
        run_reference_arm(a)
        return

    import torch
    import torch.distributed as dist

    from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, init_params, mp_params, nccl_unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = a.gpus
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = workload(n, a.scaling, a.mode)
    if a.elements:
        wl["E"] = a.elements
        wl["unique_nodes"] = (a.elements * P_ORDER + 1) ** 3
    H, M, k = wl["H"], wl["M"], wl["k"]

    uid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    torch.cuda.set_device(local)
    t0 = time.time()
    g = build_rank_graph(wl["E"], wl["p"], n, rank, "verify")
    t_graph = time.time() - t0
    cfg = GnnConfig("bench", H, M, k, mode=wl["mode"])
    eng = Engine(local, rank, n, uid)
    eng.upload_graph(g)
    eng.configure(cfg)
    eng.upload_params(mp_params(cfg, init_params(cfg, 0)))
    eng.set_option("halo_overlap", a.halo_overlap)
    if a.halo_sm_reserve >= 0:
        eng.set_option("halo_sm_reserve", a.halo_sm_reserve)
    if a.fact >= 0:
        eng.set_option("edge_factorized", a.fact)
    for kv in a.opt:
        k_, v_ = kv.split("=", 1)
        eng.set_option(k_, int(v_))
    eng.synthetic_inputs(seed=1234)
    stream = torch.cuda.ExternalStream(eng.stream_ptr)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(a.warmup):
        eng.step_device()
    barrier()
    clocks = Clocks(local) if not a.profile else None
    eng.kernel_timing(True)
    eng.launch_count(reset=True)
    eng.halo_bytes(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    for _ in range(a.steps):
        eng.step_device()
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1) / a.steps
    launches = eng.launch_count()  # all of the repo's kernel launches inside the timed region (K steps)
    ktimes = eng.kernel_times()
    halo_bytes = eng.halo_bytes() // a.steps
    eng.kernel_timing(False)
    clk = clocks.stop() if clocks else None
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = wl["unique_nodes"] * M / (ms_max / 1e3)
    sum_local = g.num_local  # the reference harness's count: coincident copies included (harness.cpp:316-321)
    if world > 1:
        t = torch.tensor([float(g.num_local)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        sum_local = int(t.item())

    # ---- halo time share (exposed and raw), N > 1 with an exchange.
    # raw: pack + exchange + sync kernels of the serial schedule (compute
    # stream, CUDA events) / serial step; exposed: extra step time of the
    # default (overlapped) schedule over the same step without the exchange
    # (mode none: the inconsistent baseline of configs[4]), both max over ranks.
    halo = None
    if world > 1 and wl["mode"] != "none" and not a.profile:
        def timed_steps(k_steps):
            barrier()
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0_.record(stream)
            for _ in range(k_steps):
                eng.step_device()
            e1_.record(stream)
            barrier()
            t_ = torch.tensor([e0_.elapsed_time(e1_) / k_steps], dtype=torch.float64)
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
            return float(t_.item())
        k2 = max(2, a.steps // 2)
        eng.set_option("halo_overlap", 0)
        eng.step_device()
        eng.kernel_timing(True)
        t_serial = timed_steps(k2)
        h_ms = eng.kernel_times()["halo"][0] / k2
        eng.kernel_timing(False)
        hm = torch.tensor([h_ms], dtype=torch.float64)
        dist.all_reduce(hm, op=dist.ReduceOp.MAX)
        eng.set_option("halo_overlap", a.halo_overlap)
        eng.configure(GnnConfig("bench", H, M, k, mode="none"))
        eng.step_device()
        t_none = timed_steps(k2)
        eng.configure(cfg)
        halo = {"halo_raw_share": float(hm.item()) / t_serial, "halo_raw_ms_per_step": float(hm.item()),
                "serial_ms_per_step": t_serial, "none_ms_per_step": t_none,
                "halo_exposed_share": max(0.0, (ms_max - t_none) / ms_max),
                "halo_exposed_ms_per_step": ms_max - t_none,
                "basis": "raw = pack + exchange + sync kernels of the serial schedule (CUDA events, compute stream) "
                         "/ serial step; exposed = (default-schedule step - same step with mode none) / "
                         "default-schedule step; max over ranks"}

    # ---- roofline of the dominant kernel class (live CUDA-event durations)
    per_launch = {c: (t / max(nl_, 1), nl_) for c, (t, nl_) in ktimes.items()}
    step_share = {c: t / a.steps / ms for c, (t, _) in ktimes.items()}
    fact_used = ktimes.get("edge_proj", (0.0, 0))[1] > 0  # factorised edge kernels ran
    ef = edge_flops_fact(H, k) if fact_used else edge_flops(H, k)
    flops = {"edge_bwd": g.num_edges * 2 * ef, "edge_fwd": g.num_edges * ef,
             "node_bwd": g.num_local * 2 * node_flops(H, k), "node_fwd": g.num_local * node_flops(H, k)}
    dom = max(flops, key=lambda c: ktimes[c][0])
    peaks = json.load(open(ROOT / "MEASURED_PEAKS.json")) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    bf16 = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops") or 1590.0
    tf32_peak = bf16 / 2.0
    avg_ms = per_launch[dom][0]
    achieved = flops[dom] / (avg_ms / 1e3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.load(open(prof)).get("kernels", {}).get(dom, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                "frac": achieved / tf32_peak, "traffic": traffic, "kernel": dom,
                "peak_basis": "dense TF32 = 1/2 of measured sustained bf16 (MEASURED_PEAKS.json)",
                "flops_per_launch": flops[dom], "ms_per_launch": avg_ms,
                "pipe": ("tcgen05 kind::tf32 3xTF32 (3 tensor products per algorithmic product; the backward "
                         "kernel also recomputes the forward: algorithmic flops exclude both)"),
                "edge_flops_basis": ("factorised: 2H^2(2+k) per edge and direction (the x_src / x_dst blocks of "
                                     "the input linear run at node level)") if fact_used else
                ("3-segment: 2H^2(4+k) per edge and direction")}

    # ---- HBM-bound kernels: algorithmic bytes per step / live kernel time per step
    hbm_peak = peaks.get("hbm_gbs") or 7700.0
    per_layer_bytes = {
        # e' rows + 1/d per in-edge read, a row written, segment bounds
        "aggregate": g.num_edges * (H * 4 + 4) + g.rows * (H * 4 + 8),
        # d_src (twin slot) + d_dst rows and the twin index per in-edge, dx_node read, dx written
        "dx_gather": g.num_edges * (2 * H * 4 + 4) + g.num_local * H * 4 + g.rows * (H * 4 + 8),
    }
    hbm = {}
    for cls_, b in per_layer_bytes.items():
        t_step = ktimes[cls_][0] / a.steps
        if t_step > 0:
            gbs = b * M / (t_step / 1e3) / 1e9
            hbm[cls_] = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                         "bytes_per_step": b * M, "ms_per_step": t_step}

    # ---- e2e through the public C-ABI with host buffers
    e2e = None
    if not a.no_e2e and not a.profile:
        e2e = run_e2e(a, eng, g, cfg, stream, barrier, world, dist, torch, wl)

    # ---- full training step on the device, supplementary
    train = None
    if not a.no_train_step and not a.profile:
        train = run_train_step(a, eng, g, cfg, stream, barrier, world, dist, torch, wl)

    # ---- CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and n == 1 and not a.no_cpu_baseline and not a.profile:
        try:
            res = cpu_reference_sample(1, a.ref_elements)
            cpu = {k2: res[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": a.steps, "warmup": a.warmup,
                "ms_per_step": ms_max, "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded by global id; random-init weights init_params seed 0)",
                "config": config_dict(wl, n), "e2e": e2e, "gpu_launches": launches,
                "gpu_launches_per_step": launches // a.steps, "roofline": roofline,
                "cpu_baseline": cpu, "clocks": clk, "train_step": train, "hbm_kernels": hbm,
                "kernel_share": {c: round(v, 4) for c, v in step_share.items()},
                "halo_bytes_per_step_rank0": halo_bytes,
                "halo_overlap": bool(a.halo_overlap and n > 1 and wl["mode"] != "none"),
                "halo_sm_reserve": a.halo_sm_reserve,
                **(halo or {}),
                "sum_local_rows": sum_local,
                "harness_layer_rows_per_s": sum_local * M / (ms_max / 1e3),
                "graph_build_s": round(t_graph, 3),
                "nodes_per_sec_per_iteration": wl["unique_nodes"] / (ms_max / 1e3)}
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def run_train_step(a, eng, g, cfg, stream, barrier, world, dist, torch, wl, steps=2):
    """hgnn_train_step (encoders + MP stack + decoder + consistent loss +
    gradient AllReduce + Adam), device time per step, max over ranks.
    Synthetic features of the reference shapes: F_x = 3, F_e = 7, autoencoding."""
    from paper_2410_01657_b200 import init_params
    eng.model_configure(3, 7, 3)
    eng.model_params_upload(init_params(cfg, 0))
    rng = np.random.default_rng(3)
    node = np.sin(0.37 * g.global_ids[:, None] + np.arange(3)[None, :])
    edge = rng.uniform(-1, 1, (g.num_edges, 7))
    eng.model_set_data(node, edge, None)
    eng.train_step()  # warm-up
    barrier()
    eng.kernel_timing(True)
    k0 = eng.kernel_times()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    losses = [eng.train_step() for _ in range(steps)]
    ev1.record(stream)
    barrier()
    k1 = eng.kernel_times()
    eng.kernel_timing(False)
    ms = ev0.elapsed_time(ev1) / steps
    share = {c: round((k1[c][0] - k0[c][0]) / steps / ms, 4) for c in k1}
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"ms_per_step": ms, "unique_nodes_per_s": wl["unique_nodes"] / (ms / 1e3), "steps": steps,
            "losses": losses, "kernel_share": share, "api": "hgnn_train_step (model.cpp:569-579 on the device)"}


def run_e2e(a, eng, g, cfg, stream, barrier, world, dist, torch, wl):
    H = cfg.hidden_dim
    rows, ne = g.rows, g.num_edges

    def pinned(shape):
        try:
            t = torch.empty(shape, dtype=torch.float64, pin_memory=True)
            return t.numpy(), True
        except Exception:
            return np.empty(shape, dtype=np.float64), False

    x0, p1 = pinned((rows, H))
    e0, p2 = pinned((ne, H))
    dx, p3 = pinned((rows, H))
    # outputs the reference's callers consume: x_M (decoder input), dx0 / de0
    # (encoder adjoints), MP-layer gradients; pinned and reused every step
    n_par = len(eng.grads())
    xo, p4 = pinned((rows, H))
    dx0, p5 = pinned((rows, H))
    de0, p6 = pinned((ne, H))
    gr, p7 = pinned((n_par,))
    rng = np.random.default_rng(5)
    blk = rng.uniform(-1, 1, (4096, H))
    for arr in (x0, e0, dx):
        for o in range(0, arr.shape[0], 4096):
            m = min(4096, arr.shape[0] - o)
            arr[o:o + m] = blk[:m]
    dx *= 1e-3
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.nmp_forward(x0, e0, out=(xo, None))  # warm-up (allocations, page-in)
    eng.nmp_backward(dx, out=(dx0, de0, gr))
    barrier()
    ev0.record(stream)
    for _ in range(a.e2e_steps):
        eng.nmp_forward(x0, e0, out=(xo, None))
        eng.nmp_backward(dx, out=(dx0, de0, gr))
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1) / a.e2e_steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": wl["unique_nodes"] * cfg.num_mp_layers / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int((2 * rows + ne) * H * 8),
            "d2h_bytes_per_step": int((2 * rows + ne) * H * 8 + n_par * 8),
            "ms_per_step": ms, "pinned": bool(p1 and p2 and p3 and p4 and p5 and p6 and p7), "steps": a.e2e_steps,
            "api": "hgnn_mp_forward + hgnn_mp_backward (fp64 host, reference edge-id order): "
                   "x0, e0, dx_M in; x_M, dx0, de0, MP-layer grads out"}


if __name__ == "__main__":
    main()
