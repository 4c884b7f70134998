#!/usr/bin/env python
"""TurboAttention (arXiv 2412.08585) hot-path benchmark on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the whole hot path over one batch of the config
BASELINE.json's metric is quoted on (configs[1]: Llama-3-8B attention shape,
32 query / 8 KV heads, d = 128, prefill N = 4096, batch 8, causal):
  turbo_quantize_kv(PREFILL)  stage-1 INT8 K/V + stage-2 INT4/INT2 cache   (a1, a2)
  turbo_attention_prefill     tcgen05 INT8 QK^T / PV with SAS softmax     (a1 Q, a4-a8)
  turbo_quantize_kv(APPEND)   one decode token into the INT8 buffer       (a3)
  turbo_attention_decode      split-KV decode over the fresh cache + LSE  (a9, a10)
`value` = prefill attention ops (4 d per unmasked (query, key) pair, 2 ops
per MAC x 2 contractions) / step time, whole job over all ranks.  A second
object `decode` measures configs[2] (Phi-3-medium shape, 40/10 heads, batch
64 at 32k context, mixed INT4/INT2 cache): KV GB/s and tokens/s.

Multi-GPU (torchrun): every rank runs its own batch (weak scaling, no data-path
collective: the prefill is partitioned by (batch, KV head)).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASE_METRIC = "attention TOPS (prefill) and KV GB/s + tokens/s (decode) at 1/2/4/8 B200 vs roofline"
CFG_PREFILL = dict(B=8, N=4096, Hq=32, Hkv=8, d=128)
CFG_DECODE = dict(B=64, N=32768, Hq=40, Hkv=10, d=128)


def prefill_ops(B, N, Hq, d, causal=True):
    pairs = N * (N + 1) // 2 if causal else N * N
    return 4.0 * d * pairs * B * Hq


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        m = json.load(open(path))
        return dict(hbm=m["hbm_gbs"], bf16=m["bf16_tflops"], bf16_sus=m.get("bf16_tflops_sustained"),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


def traffic_per_launch(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the
    committed `ncu --set full` capture summary (profiles/traffic.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)[kernel]["bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


class Clocks:
    """SM clock + throttle-reason sampler over the timed region (B200_PROFILING.md
    clocks line), polled through NVML every 50 ms from a thread.  (nvidia-smi -lms
    block-buffers its stdout, so a terminated sampler can leave an empty file.)"""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu):
        import threading

        self.rows, self.stop_ev, self.t = [], threading.Event(), None
        try:
            import pynvml as nv

            nv.nvmlInit()
            phys = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
            idx = int(phys[gpu]) if len(phys) > gpu and phys[gpu].strip().isdigit() else gpu
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            masks = [(n, getattr(nv, c)) for n, c in self.REASONS]

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), [n for n, m in masks if r & m]))
                    except Exception:
                        pass
                    self.stop_ev.wait(0.05)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None

    def stop(self):
        if self.t is None:
            return None
        self.stop_ev.set()
        self.t.join()
        if not self.rows:
            return None
        reasons = sorted({n for _, rs in self.rows for n in rs})
        load = [s for s, _ in self.rows if s > 300] or [s for s, _ in self.rows]
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": float(self.max_mhz), "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------------------- ours
def bind_host_to_gpu(device):
    """Pin this process to the CPUs of the GPU's NUMA node so the pinned host
    buffers of the e2e leg are first-touched on the node next to its PCIe root
    (a remote node roughly halves H2D/D2H bandwidth).  Best effort."""
    import torch

    try:
        pr = torch.cuda.get_device_properties(device)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return bdf
    except (OSError, ValueError, RuntimeError):
        pass
    return None


def run_ours(args, rank, world, device):
    import torch

    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import synth

    torch.cuda.set_device(device)
    bind_host_to_gpu(device)
    c = CFG_PREFILL
    B, N, Hq, Hkv, d = c["B"], c["N"], c["Hq"], c["Hkv"], c["d"]
    p = ta.params(head_dim=d, block_q=64, alpha_mode=0)
    q, k, v = synth.qkv_torch(1002 + 7919 * rank, B, N, Hq, Hkv, d, device=device)
    # NEXT-1 (Sec. 3.2): the headwise 2/4-bit plan of this layer from the on-device
    # head-priority planner over the prefill K/V (a per-layer calibration, outside the timed step);
    # half of the 2 Hkv (kv head, K/V) slots at 2 bits
    e_pl0, e_pl1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_pl0.record()
    prio = ta.turbo_head_priority(k, v)
    e_pl1.record()
    bits = ta.turbo_plan_bits(prio, Hkv).numpy()
    planner = {"priority_kernel_ms": round(e_pl0.elapsed_time(e_pl1), 4), "n_2bit_slots": Hkv,
               "bits_kv": bits.tolist()}
    qd, kd, vd = (x[:, 0].contiguous() for x in synth.qkv_torch(4002 + rank, B, 1, Hq, Hkv, d, device=device))
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits, device=device)
    S = args.splits
    if S is None:  # the binding's deterministic default (device-independent partition)
        S = ta.auto_splits(B, Hkv, N // 64, ta.reference_workers(Hq, Hkv, d))
    ws = torch.empty(max(ta.turbo_decode_workspace_bytes(B, Hq, Hkv, d, S), 16), dtype=torch.uint8, device=device)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=device)  # > 126 MB L2
    # read after the write: the flush's own dirty lines are written back before the step, not inside it
    flush_rd = torch.ones(64 << 20, dtype=torch.float32, device=device)  # 256 MB
    st = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(qq, kk, vv, qdd, kdd, vdd, evs=None, bufs=None):
        # bufs: preallocated outputs (the e2e loop double-buffers them; the allocator
        # would otherwise cudaMalloc -- and synchronise -- while copies are in flight)
        if evs:
            evs[0].record(st)
        k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, kk, vv, out=bufs["kv"] if bufs else None)
        if evs:
            evs[1].record(st)
        o, lse = ta.turbo_attention_prefill(p, qq, k1, v1t, k1s, v1s, causal=True,
                                            o=bufs["o"] if bufs else None, lse=bufs["lse"] if bufs else None)
        if evs:
            evs[2].record(st)
        ta.turbo_quantize_kv(p, cache, kdd, vdd, mode=1)
        od, _, lsed = ta.turbo_attention_decode(p, cache, qdd, n_splits=S, workspace=ws,
                                                o=bufs["od"] if bufs else None, lse=bufs["lsed"] if bufs else None)
        if evs:
            evs[3].record(st)
        return o, lse, od, lsed

    # our kernels per step: quantize_kv PREFILL (the TMA kernel; + quant_tail_kernel when N is not a whole number of
    # B_c blocks -- its a_univ reset is a cudaMemsetAsync), the prefill, APPEND (append + counters), decode (+ combine)
    launches_per_step = (1 if N % 64 == 0 else 2) + 1 + 2 + (2 if S > 1 else 1)
    clk = Clocks(device) if rank == 0 else None  # sampler runs through the soak and the timed steps
    for _ in range(args.warmup):
        step(q, k, v, qd, kd, vd)
    torch.cuda.synchronize()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 0.7:  # untimed soak: clocks/power settle, sampler is live
        step(q, k, v, qd, kd, vd)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    evs = [[ev() for _ in range(4)] for _ in range(args.steps)]
    torch.cuda._sleep(1000)  # (first use of the between-step kernels before the timed loop: lazy module loading)
    flush.zero_()
    flush_rd.sum()
    torch.cuda.synchronize()
    for i in range(args.steps):
        # ~0.5 ms of GPU work before each step, outside its events: the host enqueues the step while it runs, so
        # no step's events include host launch latency (Python / the NVML clock sampler holding the GIL)
        torch.cuda._sleep(1_000_000)
        flush.zero_()  # L2 flush between timed steps (outside the events): write 512 MB, then read 256 MB
        flush_rd.sum()
        step(q, k, v, qd, kd, vd, evs[i])
    torch.cuda.synchronize()
    clocks = clk.stop() if clk else None
    t_quant = [e[0].elapsed_time(e[1]) for e in evs]
    t_prefill = [e[1].elapsed_time(e[2]) for e in evs]
    t_dec = [e[2].elapsed_time(e[3]) for e in evs]
    t_step = [e[0].elapsed_time(e[3]) for e in evs]
    total_ms = sum(t_step)
    if world > 1:
        t = torch.tensor([total_ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = t.item()
    ms_step = total_ms / args.steps
    ops = prefill_ops(B, N, Hq, d)
    value = world * ops * args.steps / (total_ms * 1e-3) / 1e12

    # ---- end to end through the public API: pinned host inputs -> device -> host result.
    # Every step copies its inputs in and its outputs out; the copies run on their own
    # streams (H2D and D2H copy engines, full-duplex PCIe) and overlap the neighbouring
    # steps' compute, with double-buffered device tensors -- how a serving loop would run.
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    hqd, hkd, hvd = (x.cpu().pin_memory() for x in (qd, kd, vd))
    ho = torch.empty(q.shape, dtype=torch.float16).pin_memory()
    hlse = torch.empty((B, Hq, N), dtype=torch.float32).pin_memory()
    hod = torch.empty(qd.shape, dtype=torch.float16).pin_memory()
    dins = [[torch.empty_like(x) for x in (q, k, v, qd, kd, vd)] for _ in range(2)]
    tcb = N // 64
    douts = [{"kv": (torch.empty((B, Hkv, N, d), dtype=torch.float16, device=device),
                     torch.empty((B, Hkv, tcb, d, 64), dtype=torch.float16, device=device),
                     torch.empty((B, Hkv, tcb), dtype=torch.float32, device=device),
                     torch.empty((B, Hkv, tcb), dtype=torch.float32, device=device)),
              "o": torch.empty_like(q), "lse": torch.empty((B, Hq, N), dtype=torch.float32, device=device),
              "od": torch.empty_like(qd), "lsed": torch.empty((B, Hq), dtype=torch.float32, device=device)}
             for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(device), torch.cuda.Stream(device)
    e2e_steps = max(4, min(args.steps, 32))  # amortises the pipeline fill and drain
    e0, e1 = ev(), ev()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0.record(st)
    s_in.wait_stream(st)
    s_out.wait_stream(st)
    in_ready, in_free, out_done = [None] * e2e_steps, [None] * e2e_steps, [None] * e2e_steps
    outs = [None] * e2e_steps
    for i in range(e2e_steps):
        buf = dins[i % 2]
        with torch.cuda.stream(s_in):
            if i >= 2:
                s_in.wait_event(in_free[i - 2])  # step i-2 has consumed this input buffer
            for dst, src in zip(buf, (hq, hk, hv, hqd, hkd, hvd)):
                dst.copy_(src, non_blocking=True)
            in_ready[i] = torch.cuda.Event()
            in_ready[i].record(s_in)
        st.wait_event(in_ready[i])
        if i >= 2:
            st.wait_event(out_done[i - 2])  # the outputs of step i-2 have left the device
        outs[i] = step(*buf, bufs=douts[i % 2])
        in_free[i] = torch.cuda.Event()
        in_free[i].record(st)
        with torch.cuda.stream(s_out):
            s_out.wait_event(in_free[i])
            o, lse, od, _ = outs[i]
            ho.copy_(o, non_blocking=True)
            hlse.copy_(lse, non_blocking=True)
            hod.copy_(od, non_blocking=True)
            out_done[i] = torch.cuda.Event()
            out_done[i].record(s_out)
    st.wait_stream(s_out)
    e1.record(st)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = t.item()
    h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv, hqd, hkd, hvd))
    d2h = sum(x.numel() * x.element_size() for x in (ho, hlse, hod))
    # this host's pinned-copy bandwidth (the e2e figure is PCIe-bound and varies between hosts)
    probe = {}
    try:
        hb = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
        db = torch.empty(256 << 20, dtype=torch.uint8, device=device)
        for name, fn in (("h2d_gbs", lambda: db.copy_(hb, non_blocking=True)),
                         ("d2h_gbs", lambda: hb.copy_(db, non_blocking=True))):
            fn()
            best = float("inf")
            for _ in range(3):
                p0, p1 = ev(), ev()
                p0.record(st)
                fn()
                p1.record(st)
                torch.cuda.synchronize()
                best = min(best, p0.elapsed_time(p1))
            probe[name] = round((256 << 20) / (best * 1e-3) / 1e9, 1)
        del hb, db
    except RuntimeError:
        pass
    e2e = {"value": world * ops * e2e_steps / (e2e_ms * 1e-3) / 1e12, "unit": "TOPS", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / e2e_steps, "steps": e2e_steps,
           "pcie_probe": probe}

    pk = peaks()
    int8_peak = 2.0 * pk["bf16"]  # dense int8 = 2 x dense bf16 (nominal 4.5 vs 2.25 PF), burst
    pre_ms = statistics.mean(t_prefill)
    achieved = ops / (pre_ms * 1e-3) / 1e12
    # context: a plain INT8 GEMM (cuBLASLt through torch._int_mm, 8192^3, best of 10) on this GPU; the
    # roofline keeps the contract's peak (2 x the measured bf16 burst, the nominal int8 / bf16 ratio)
    int8_gemm = None
    try:
        ga = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device=device)
        gb = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device=device).t()
        torch._int_mm(ga, gb)
        best = float("inf")
        for _ in range(10):
            g0, g1 = ev(), ev()
            g0.record(st)
            torch._int_mm(ga, gb)
            g1.record(st)
            torch.cuda.synchronize()
            best = min(best, g0.elapsed_time(g1))
        int8_gemm = round(2 * 8192 ** 3 / (best * 1e-3) / 1e12, 1)
        del ga, gb
    except (RuntimeError, AttributeError):
        pass
    roof = {"bound": "tensor", "kernel": "prefill_kernel<128> (turbo_attention_prefill)", "achieved": round(achieved, 1),
            "peak": round(int8_peak, 1), "unit": "TFLOP/s", "frac": round(achieved / int8_peak, 4),
            "traffic": traffic_per_launch("prefill_kernel"), "peak_source": f"2 x bf16 burst {pk['bf16']} TF/s, {pk['src']}",
            "share_of_step": round(pre_ms / statistics.mean(t_step), 3),
            "int8_gemm_tops_measured": int8_gemm,
            # QK^T (2d ops / score element) and P'.V hi + lo (2 x 2d) all run as kind::f16 at the bf16/fp16 rate:
            # 4d reported ops per 6d tensor flops
            "tensor_ceiling_of_mma_mix": round(4.0 / 6.0 * pk["bf16"], 1)}
    # The bound that actually binds: the FP32 (FMA) pipe running the bit-exact SAS mix.
    # Unit counts: 4 SMSPs x 32 lanes x 2 elements per packed FMA-pipe instruction at 0.5 instr / clk
    # = 128 element-operations / clk / SM; the pinned arithmetic needs 13 per score element (x, d,
    # floor, floor - magic, fraction, Horner x 3, LUT product, row sum, P code, P' hi, P' lo), and a
    # score element carries 4 d = 512 ops.  Clock: the median SM clock under load.
    sm_hz = (clocks or {}).get("sm_mhz") or 1965.0
    alu_peak = 148 * 128 / 13 * sm_hz * 1e6 * 4 * d / 1e12
    roof["alu_bound"] = {"bound": "alu", "achieved": round(achieved, 1), "peak": round(alu_peak, 1), "unit": "TOPS",
                         "frac": round(achieved / alu_peak, 4),
                         "peak_source": f"148 SMs x 128 FP32-pipe element-ops/clk / 13 per score element x "
                                        f"{sm_hz:.0f} MHz x 512 ops per element (DESIGN.md 7)",
                         "measured_mix_ceiling_tops": 745.0}
    # quantize_kv (a1/a2) as its own HBM-bound kernel: FP16 K, V in; k1 and v1t (stage-1 codes carried in FP16), records,
    # scales out
    q_ms = statistics.mean(t_quant)
    rec_b = B * Hkv * (N // 64) * sum(2 * d + 64 * d * int(bits[h][kd]) // 8 for h in range(Hkv) for kd in range(2)) // Hkv
    q_bytes = 2 * B * N * Hkv * d * 2 + B * N * Hkv * d * 2 + B * N * Hkv * d * 2 + rec_b + 2 * B * Hkv * (N // 64) * 8
    quant = {"ms": round(q_ms, 4), "ms_median": round(statistics.median(t_quant), 4), "ms_min": round(min(t_quant), 4),
             "ms_first": round(t_quant[0], 4), "bytes": q_bytes, "gbs": round(q_bytes / (q_ms * 1e-3) / 1e9, 1),
             "frac_hbm": round(q_bytes / (q_ms * 1e-3) / 1e9 / pk["hbm"], 4)}
    # ---- deviation from exact attention (Eq. 2), reported separately (north_star):
    # sampled (b, q head) units and query rows of configs[1], both alpha modes (after the timed region)
    deviation = None
    if rank == 0 and not args.no_deviation:
        o0 = step(q, k, v, qd, kd, vd)[0]
        p1 = ta.params(head_dim=d, block_q=64, alpha_mode=1)
        k1_, v1t_, k1s_, v1s_ = ta.turbo_quantize_kv(p1, cache, k, v)
        o1, _ = ta.turbo_attention_prefill(p1, q, k1_, v1t_, k1s_, v1s_, causal=True)
        units = [(0, 0), (1, 5), (3, 13), (5, 22), (7, 31)]
        rows = sorted(set(range(7, N, 29)) | {N - 1})
        deviation = {"prefill_configs1": dict(
            units=f"(b, q head) {units}, {len(rows)} query rows each (every 29th + the last)",
            **deviation_prefill(p, q, k, v, {0: o0, 1: o1}, units, rows))}
        # NEXT-2 variants, each with its kernel speed and its deviation on the same units:
        #  * prefill P scale per row x B_c block (Alg. 2's granularity) instead of per B_r x B_c
        #    tile (Alg. 1);
        #  * first-stage scales stored in FP16 (R-29);
        #  * the SAS polynomial in FP16 (R-30);
        #  * B_c = 128 (the block-size ablation, Table 3): its own cache and prefill operands.
        variants = {}
        g0, g1 = ev(), ev()
        for name, kw in (("prefill_p_scale_per_row", dict(p_scale_rows=1)),
                         ("first_stage_scales_fp16", dict(scale_fp16=1)),
                         ("sas_polynomial_fp16", dict(sas_fp16=1)),
                         ("block_kv_128", dict(block_kv=128))):
            pv = ta.params(head_dim=d, block_q=64, alpha_mode=0, **kw)
            cv = cache if pv.block_kv == 64 else ta.KVCache(B, Hkv, d, max_blocks=N // pv.block_kv + 2, bits=bits,
                                                             block_kv=pv.block_kv, device=device)
            k1_, v1t_, k1s_, v1s_ = ta.turbo_quantize_kv(pv, cv, k, v)
            ov, lv = ta.turbo_attention_prefill(pv, q, k1_, v1t_, k1s_, v1s_, causal=True)
            g0.record(st)
            for _ in range(10):
                ta.turbo_attention_prefill(pv, q, k1_, v1t_, k1s_, v1s_, causal=True, o=ov, lse=lv)
            g1.record(st)
            torch.cuda.synchronize()
            v_ms = g0.elapsed_time(g1) / 10
            variants[name] = {
                "kernel_ms": round(v_ms, 4), "tops": round(ops / (v_ms * 1e-3) / 1e12, 1),
                "deviation_alpha_mode_0": deviation_prefill(pv, q, k, v, {0: ov}, units, rows)["alpha_mode_0"]}
            del ov, lv, k1_, v1t_, k1s_, v1s_, cv
        deviation["variants"] = variants
        del o0, o1
    result = dict(value=value, ms_step=ms_step, e2e=e2e, roofline=roof, clocks=clocks, quantize_kv=quant,
                  deviation=deviation,
                  planner=planner,
                  launches=launches_per_step * args.steps,
                  breakdown_ms={"quantize_kv_prefill": round(statistics.mean(t_quant), 4),
                                "attention_prefill": round(pre_ms, 4),
                                "append+decode": round(statistics.mean(t_dec), 4)})
    del hq, hk, hv, ho, hlse, dins, douts, outs, q, k, v, flush, flush_rd, cache
    torch.cuda.empty_cache()
    if not args.no_decode:
        result["decode"] = bench_decode(args, rank, world, device, pk)
    return result


def decode_bytes(B, Hkv, d, nblk, nbuf, bits, Hq, bc=64):
    """Algorithmic HBM bytes of one decode step: block records (s_int, z_int,
    packed codes), parent scales, buffer rows, q in, o/lse out (nblk blocks of bc tokens)."""
    per_bh = 0
    for h in range(Hkv):
        for kind in range(2):
            per_bh += nblk * (2 * d + bc * d * int(bits[h][kind]) // 8 + 4) + nbuf * d + 4
    return B * per_bh + B * Hq * d * 2 * 2 + B * Hq * 4


def bench_decode(args, rank, world, device, pk):
    import torch

    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import synth

    c = CFG_DECODE
    B, N, Hq, Hkv, d = c["B"], c["N"], c["Hq"], c["Hkv"], c["d"]
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, alpha_mode=0)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 4, bits=bits, device=device)
    _, k, v = synth.qkv_torch(3003 + rank, B, N, Hkv, Hkv, d, device=device)
    ta.turbo_quantize_kv(p, cache, k, v)  # builds the 32k-token compressed cache
    dev_units = [(0, 0), (13, 7), (40, 22), (63, 39)]  # (b, q head) sampled for the deviation report
    G = Hq // Hkv
    host_kv = {(b, h // G): (k[b, :, h // G].float().cpu().numpy(), v[b, :, h // G].float().cpu().numpy())
               for b, h in dev_units}
    del k, v
    torch.cuda.empty_cache()
    S = args.decode_splits
    if S is None:  # the binding's deterministic default (device-independent partition)
        S = ta.resolve_splits(None, B, Hq, cache)
    ws = torch.empty(max(ta.turbo_decode_workspace_bytes(B, Hq, Hkv, d, S), 16), dtype=torch.uint8, device=device)
    toks = [tuple(x[:, 0].contiguous() for x in synth.qkv_torch(6000 + i, B, 1, Hq, Hkv, d, device=device))
            for i in range(args.warmup + args.steps)]
    st = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for i in range(args.warmup):
        qd, kd, vd = toks[i]
        ta.turbo_quantize_kv(p, cache, kd, vd, mode=1)
        ta.turbo_attention_decode(p, cache, qd, n_splits=S, workspace=ws)
    torch.cuda.synchronize()
    evs = [[ev() for _ in range(3)] for _ in range(args.steps)]
    for i in range(args.steps):
        qd, kd, vd = toks[args.warmup + i]
        evs[i][0].record(st)
        ta.turbo_quantize_kv(p, cache, kd, vd, mode=1)
        evs[i][1].record(st)
        ta.turbo_attention_decode(p, cache, qd, n_splits=S, workspace=ws)
        evs[i][2].record(st)
    torch.cuda.synchronize()
    deviation = None
    if rank == 0 and not args.no_deviation:
        import numpy as np

        qd = synth.qkv_torch(6999, B, 1, Hq, Hkv, d, device=device)[0][:, 0].contiguous()
        outs = {}
        for mode in (0, 1):
            pm = ta.params(head_dim=d, alpha_mode=mode)
            outs[(mode, S)] = ta.turbo_attention_decode(pm, cache, qd, n_splits=S)[0].float().cpu().numpy()
            outs[(mode, 1)] = ta.turbo_attention_decode(pm, cache, qd, n_splits=1)[0].float().cpu().numpy()
        qh = qd.float().cpu().numpy()
        refs, vr = [], []
        for b, h in dev_units:
            kk, vv = host_kv[(b, h // G)]
            ka = np.concatenate([kk] + [toks[i][1][b, h // G].float().cpu().numpy()[None] for i in range(len(toks))])
            va = np.concatenate([vv] + [toks[i][2][b, h // G].float().cpu().numpy()[None] for i in range(len(toks))])
            refs.append(exact_attention(qh[b, h][None], ka, va, 1.0 / math.sqrt(d))[0])
            vr.append(va)
        v_rms = float(np.sqrt(np.mean(np.concatenate(vr) ** 2)))
        ref = np.stack(refs)
        pick = lambda o: np.stack([o[b, h] for b, h in dev_units])  # noqa: E731
        deviation = {"units": f"(b, q head) {dev_units}, one query after {cache.n_tokens} tokens; "
                              f"(K, V) bits {[tuple(int(x) for x in bits[h // G]) for _, h in dev_units]}",
                     "default_splits": S}
        for mode in (0, 1):
            deviation[f"alpha_mode_{mode}"] = {
                "unsplit_vs_exact": dev_stats(pick(outs[(mode, 1)]), ref, v_rms),
                "split_vs_exact": dev_stats(pick(outs[(mode, S)]), ref, v_rms),
                "split_vs_unsplit_rel_l2": dev_stats(outs[(mode, S)], outs[(mode, 1)], 1.0)["rel_l2"]}
    t_dec = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    t_step = statistics.mean(e[0].elapsed_time(e[2]) for e in evs)
    ntok = cache.n_tokens
    nblk, nbuf = ntok // 64, ntok % 64
    byt = decode_bytes(B, Hkv, d, nblk, nbuf, bits, Hq)
    gbs = byt / (t_dec * 1e-3) / 1e9
    return {"deviation": deviation,
            "config": "Phi-3-medium attention (40 Q / 10 KV heads, d=128), batch 64, 32k context, mixed INT4/INT2",
            "n_splits": S, "kv_bytes_per_step": byt, "decode_kernel_ms": round(t_dec, 4),
            "step_ms_append_plus_decode": round(t_step, 4), "kv_gbs": round(gbs, 1),
            "tokens_per_s": round(world * B / (t_step * 1e-3), 1),
            "tokens_per_s_40_layers": round(world * B / (t_step * 1e-3) / 40, 1),  # Phi-3-medium: 40 attention layers
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": pk["hbm"], "unit": "GB/s",
                         "traffic": traffic_per_launch("decode_kernel"),
                         "frac": round(gbs / pk["hbm"], 4), "peak_source": pk["src"]}}


# --------------------------------------------------------------------------- deviation from exact attention
def exact_attention(q, k, v, scale, q_pos=None):
    """Eq. 2 in FP64: softmax(q k^T scale) v for query rows q [n, d] at absolute
    positions q_pos (causal: keys 0..q_pos; None: all keys visible).  The plain definition, no
    quantisation, no SAS -- the reference the method's deviation is reported against."""
    import numpy as np

    q, k, v = (np.asarray(x, np.float64) for x in (q, k, v))
    s = (q @ k.T) * scale
    if q_pos is not None:
        s = np.where(np.arange(k.shape[0])[None, :] <= np.asarray(q_pos)[:, None], s, -np.inf)
    s -= s.max(axis=1, keepdims=True)
    w = np.exp(s)
    return (w / w.sum(axis=1, keepdims=True)) @ v


def dev_stats(o, ref, v_rms):
    import numpy as np

    o, ref = np.asarray(o, np.float64), np.asarray(ref, np.float64)
    return {"rel_l2": float(np.linalg.norm(o - ref) / np.linalg.norm(ref)),
            "max_abs": float(np.abs(o - ref).max()), "max_abs_over_rms_v": float(np.abs(o - ref).max() / v_rms),
            "rms_err_over_rms_v": float(np.sqrt(np.mean((o - ref) ** 2)) / v_rms)}


def deviation_prefill(p_mode, q, k, v, o_by_mode, units, rows):
    """configs[1] prefill: the GPU output of sampled (b, q head) units and query rows against Eq. 2,
    per alpha mode (R-15)."""
    import numpy as np

    G = q.shape[2] // k.shape[2]
    d = q.shape[3]
    out = {}
    for mode, o in o_by_mode.items():
        os_, rs, vr = [], [], []
        for b, h in units:
            qh = q[b, :, h].float().cpu().numpy()
            kh, vh = k[b, :, h // G].float().cpu().numpy(), v[b, :, h // G].float().cpu().numpy()
            ref = exact_attention(qh[rows], kh, vh, 1.0 / math.sqrt(d), rows)
            os_.append(o[b, rows, h].float().cpu().numpy())
            rs.append(ref)
            vr.append(vh)
        out[f"alpha_mode_{mode}"] = dev_stats(np.concatenate(os_), np.concatenate(rs),
                                              float(np.sqrt(np.mean(np.concatenate(vr) ** 2))))
    return out


def trend_v_probe(device):
    """PAPER.md:921 rescale read literally (alpha_mode 0, R-15) multiplies the history by
    SAS(0) = 0.9996 per tile: a positional bias that only a value trend exposes.  One 32k-token
    sequence, V = position / N + 0.1 N(0, 1) (fp16), one query head group, K and V at 4 bits (so
    that the 2-bit reconstruction error does not hide the alpha-chain bias); decode against Eq. 2,
    unsplit and with the default split count, both alpha modes."""
    import numpy as np
    import torch

    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import synth

    N, d, Hq, Hkv = 32768 + 17, 128, 4, 1
    qx, kx, _ = synth.qkv_torch(777, 1, N, Hq, Hkv, d, device=device)
    gen = torch.Generator(device=device)
    gen.manual_seed(778)
    vx = (torch.arange(N, device=device, dtype=torch.float32)[None, :, None, None] / N
          + 0.1 * torch.randn((1, N, Hkv, d), generator=gen, device=device)).half()
    cache = ta.KVCache(1, Hkv, d, max_blocks=N // 64 + 2, bits=[[4, 4]], device=device)
    ta.turbo_quantize_kv(ta.params(head_dim=d), cache, kx.contiguous(), vx.contiguous())
    qd = qx[:, -1].contiguous()
    kh, vh = kx[0, :, 0].float().cpu().numpy(), vx[0, :, 0].float().cpu().numpy()
    ref = exact_attention(qd[0].float().cpu().numpy(), kh, vh, 1.0 / math.sqrt(d))
    S = ta.resolve_splits(None, 1, Hq, cache)
    res = {"config": f"B=1, N={N}, 4/1 heads, d=128, 4-bit K and V, V = t/N + 0.1 N(0,1), split count {S}"}
    for mode in (0, 1):
        p = ta.params(head_dim=d, alpha_mode=mode)
        o1 = ta.turbo_attention_decode(p, cache, qd, n_splits=1)[0][0].float().cpu().numpy()
        oS = ta.turbo_attention_decode(p, cache, qd, n_splits=S)[0][0].float().cpu().numpy()
        res[f"alpha_mode_{mode}"] = {"unsplit_vs_exact": dev_stats(o1, ref, float(np.sqrt(np.mean(vh ** 2))))["rel_l2"],
                                     "split_vs_exact": dev_stats(oS, ref, float(np.sqrt(np.mean(vh ** 2))))["rel_l2"],
                                     "split_vs_unsplit": dev_stats(oS, o1, 1.0)["rel_l2"]}
    return res


# --------------------------------------------------------------------------- reference (oracle)
def cpu_sample_oracle(seconds_hint=True):
    """The CPU oracle (oracle/, plain scalar C, as it stands) on a bounded sample of
    the same workload: K/V quantisation + cache build and Alg. 1 for one (batch,
    query head) unit of configs[1] (N = 4096, d = 128, causal) per host core, the
    units run concurrently on threads (ctypes releases the GIL), plus the
    single-thread time of one unit."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    from paper_2412_08585_b200 import synth

    N, d = CFG_PREFILL["N"], CFG_PREFILL["d"]
    p = O.params(d=d)
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    units = []
    for u in range(ncores):  # inputs drawn outside the timed region
        q, k, v = synth.qkv(1002 + u, 1, N, 1, 1, d)
        units.append(tuple(x[0, :, 0].astype(np.float32) for x in (q, k, v)))

    def one(u):
        q, k, v = units[u]
        ks, vs = O.Slot(p, 4, N // 64 + 1), O.Slot(p, 2, N // 64 + 1)
        ks.prefill(k)
        vs.prefill(v)
        O.prefill_head(p, q, k, v, causal=True)

    O.lib()  # build / load once, outside the timing
    t0 = time.perf_counter()
    one(0)
    dt1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=ncores) as ex:
        list(ex.map(one, range(ncores)))
    dt = time.perf_counter() - t0
    ops = prefill_ops(1, N, 1, d)
    cpu_model = None
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        pass
    return {"value": ncores * ops / dt / 1e12, "unit": "TOPS", "cores": ncores, "kind": "oracle", "cpu_model": cpu_model,
            "sample": f"{ncores} of {CFG_PREFILL['B'] * CFG_PREFILL['Hq']} (batch, head) units of configs[1] "
                      f"(quantize + cache build + Alg. 1, N={N}, d={d}, causal), one per host core on "
                      f"{ncores} threads: {dt:.2f} s; one unit single-threaded {dt1:.2f} s",
            "value_1core": ops / dt1 / 1e12, "seconds": round(dt, 3)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up state; one sample per step below
    vals, secs = [], []
    for _ in range(args.steps):
        s = cpu_sample_oracle()
        vals.append(s["value"])
        secs.append(s["seconds"])
    v = statistics.mean(vals)
    s["value"] = v
    line = {"metric": BASE_METRIC, "value": v, "unit": "TOPS", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(secs), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "impl": "reference", "config": workload_config(args),
            "cpu_baseline": s, "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args):
    c = CFG_PREFILL
    return {"workload": "configs[1]: Llama-3-8B attention shape (32 Q / 8 KV heads GQA, d=128), prefill seq 4096, "
                        "batch 8, causal, INT8 tcgen05; step = quantize_kv + prefill + append + split-KV decode",
            "global_batch": c["B"] * args.gpus, "seq_len": c["N"], "n_q_heads": c["Hq"], "n_kv_heads": c["Hkv"],
            "head_dim": c["d"], "block_q": 64, "block_kv": 64, "sas_nr": -6, "alpha_mode": 0,
            "kv_bits": "half of the (kv_head, K/V) slots 2-bit, rest 4-bit",
            "decode_splits": args.splits if args.splits is not None else "auto (binding.auto_splits)",
            "parallelism": f"(batch, kv-head) partition, {args.gpus} rank(s), no collective",
            "l2": "flushed between timed steps (512 MB write, then 256 MB read: L2 left clean)"}


# --------------------------------------------------------------------------- secondary workloads
CFG_70B = dict(B=1, N=32768, Hq=64, Hkv=8, d=128)
CFG_LONG = dict(B=16, N=128 * 1024, Hq=32, Hkv=8, d=128)


def _max_over_ranks(ms, world, device):
    import torch

    if world > 1:
        t = torch.tensor([ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = t.item()
    return ms


def run_prefill_70b(args, rank, world, device):
    """configs[3]: Llama-3-70B attention (64 Q / 8 KV heads, d=128), prefill 32k,
    batch 1; KV heads (with their query heads) partitioned over the ranks
    (strong scaling, no collective)."""
    import torch

    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import parallel, synth

    c = CFG_70B
    (k0, k1), (h0, h1) = parallel.head_shard(c["Hq"], c["Hkv"], world, rank)
    hkv, hq = k1 - k0, h1 - h0
    B, N, d = c["B"], c["N"], c["d"]
    p = ta.params(head_dim=d)
    q, k, v = synth.qkv_torch(5005 + rank, B, N, hq, hkv, d, device=device)
    cache = ta.KVCache(B, hkv, d, max_blocks=N // 64 + 1, bits=synth.head_bits_alternating(hkv), device=device)
    st = torch.cuda.current_stream()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clk = Clocks(device) if rank == 0 else None
    for i in range(args.warmup + args.steps):
        e = evs[i - args.warmup] if i >= args.warmup else None
        if e:
            e[0].record(st)
        k1_, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, k, v)
        if e:
            e[1].record(st)
        ta.turbo_attention_prefill(p, q, k1_, v1t, k1s, v1s, causal=True)
        if e:
            e[2].record(st)
    torch.cuda.synchronize()
    clocks = clk.stop() if clk else None
    ms = _max_over_ranks(sum(e[0].elapsed_time(e[2]) for e in evs), world, device) / args.steps
    ops = prefill_ops(B, N, c["Hq"], d)
    pk = peaks()
    pre_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    ach = prefill_ops(B, N, hq, d) / (pre_ms * 1e-3) / 1e12  # this rank's heads / its kernel time
    return {"value": ops / (ms * 1e-3) / 1e12, "unit": "TOPS", "ms_step": ms, "scaling": "strong", "clocks": clocks,
            "roofline": {"bound": "tensor", "kernel": "prefill_kernel<128> (rank 0)", "achieved": round(ach, 1),
                         "peak": round(2.0 * pk["bf16"], 1), "unit": "TFLOP/s",
                         "frac": round(ach / (2.0 * pk["bf16"]), 4), "traffic": None,
                         "peak_source": f"2 x bf16 burst {pk['bf16']} TF/s, {pk['src']}"},
            "config": {"workload": "configs[3]: Llama-3-70B attention shape (64 Q / 8 KV heads, d=128), prefill 32k, "
                                   "batch 1, causal; step = quantize_kv + prefill",
                       "parallelism": f"KV heads partitioned over {world} rank(s), no collective",
                       "per_rank_heads": [hq, hkv]}}


def run_prefill_chunk(args, rank, world, device):
    """NEXT-3 chunked prefill (R-28) on the configs[1] shape: a 1024-token chunk after a
    3072-token compressed prefix (B = 8, 32/8 heads, d = 128, causal); per step:
    turbo_dequantize_cache (prefix operands) + turbo_quantize_kv mode 2 (chunk) +
    turbo_attention_prefill_chunk.  Ops = 4 d x unmasked (query, key) pairs of the chunk."""
    import torch

    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import synth

    c = CFG_PREFILL
    B, Hq, Hkv, d = c["B"], c["Hq"], c["Hkv"], c["d"]
    P, Nq = 3072, 1024
    Nk = P + Nq
    p = ta.params(head_dim=d)
    q, k, v = synth.qkv_torch(6006 + rank, B, Nk, Hq, Hkv, d, device=device)
    qc, kp, vp, kc, vc = (x.contiguous() for x in (q[:, P:], k[:, :P], v[:, :P], k[:, P:], v[:, P:]))
    cache = ta.KVCache(B, Hkv, d, max_blocks=Nk // 64 + 1, bits=synth.head_bits_alternating(Hkv), device=device)
    ops_buf = ta.turbo_dequantize_cache(p, cache, Nk)
    o = torch.empty_like(qc)
    lse = torch.empty((B, Hq, Nq), dtype=torch.float32, device=device)
    st = torch.cuda.current_stream()
    tot = 0.0
    for i in range(args.warmup + args.steps):
        ta.turbo_quantize_kv(p, cache, kp, vp)  # the prefix (untimed: restores the cache to P tokens)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ta.turbo_dequantize_cache(p, cache, Nk, out=ops_buf)
        ta.turbo_quantize_kv(p, cache, kc, vc, mode=2, out=ops_buf)
        ta.turbo_attention_prefill_chunk(p, qc, *ops_buf, causal=True, o=o, lse=lse)
        e1.record(st)
        torch.cuda.synchronize()
        if i >= args.warmup:
            tot += e0.elapsed_time(e1)
    ms = _max_over_ranks(tot, world, device) / args.steps
    ops = 4.0 * d * B * Hq * sum(P + r + 1 for r in range(Nq)) * world
    return {"value": ops / (ms * 1e-3) / 1e12, "unit": "TOPS", "ms_step": ms, "scaling": "weak",
            "config": {"workload": "NEXT-3 chunked prefill (R-28): 1024-token chunk after a 3072-token compressed "
                                   "prefix, configs[1] shape (B=8, 32/8 heads, d=128), causal; step = "
                                   "dequantize_cache + quantize_kv(chunk) + prefill_chunk",
                       "parallelism": f"{world} rank(s), each its own batch, no collective"}}


def run_q_projection(args, rank, world, device):
    """NEXT-3: the Q projection with the stage-1 Q quantisation fused into its epilogue on the
    configs[1] shape (Llama-3-8B: B = 8, N = 4096, D = 4096 -> 32 heads x d = 128), then the prefill on
    the quantised query (turbo_attention_prefill_q1).  Value: projection TFLOP/s (2 T D Hq d), its
    roofline against the fp16 tensor peak (the measured bf16 burst; fp16 and bf16 share the rate)."""
    import torch

    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import synth

    c = CFG_PREFILL
    B, N, Hq, Hkv, d = c["B"], c["N"], c["Hq"], c["Hkv"], c["d"]
    D = Hq * d
    p = ta.params(head_dim=d)
    gen = torch.Generator(device=device)
    gen.manual_seed(5150 + rank)
    x = (0.5 * torch.randn((B, N, D), generator=gen, device=device)).half()
    wq = (torch.randn((Hq * d, D), generator=gen, device=device) / math.sqrt(D)).half()
    _, k, v = synth.qkv_torch(5151 + rank, B, N, Hq, Hkv, d, device=device)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=synth.head_bits_alternating(Hkv), device=device)
    ops_kv = ta.turbo_quantize_kv(p, cache, k, v)
    q1, sq, _ = ta.turbo_q_projection(p, x, wq, Hq)
    o, lse = ta.turbo_attention_prefill_q1(p, q1, sq, *ops_kv)
    st = torch.cuda.current_stream()
    t_proj = t_pre = 0.0
    clk = None
    for i in range(args.warmup + args.steps):
        if i == args.warmup:
            clk = Clocks(device) if rank == 0 else None
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        ta.turbo_q_projection(p, x, wq, Hq)
        e1.record(st)
        ta.turbo_attention_prefill_q1(p, q1, sq, *ops_kv, o=o, lse=lse)
        e2.record(st)
        torch.cuda.synchronize()
        if i >= args.warmup:
            t_proj += e0.elapsed_time(e1)
            t_pre += e1.elapsed_time(e2)
    clocks = clk.stop() if clk else None
    ms_p = _max_over_ranks(t_proj, world, device) / args.steps
    ms_a = _max_over_ranks(t_pre, world, device) / args.steps
    flops = 2.0 * B * N * D * Hq * d * world
    ops_attn = 4.0 * d * N * (N + 1) / 2 * B * Hq * world
    pk = peaks()
    ach = flops / world / (ms_p * 1e-3) / 1e12
    return {"value": flops / (ms_p * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_step": ms_p + ms_a, "scaling": "weak",
            "clocks": clocks, "dtype": "fp16",
            "roofline": {"bound": "tensor", "kernel": "q_projection_kernel<128> (turbo_q_projection)",
                         "achieved": round(ach, 1), "peak": round(pk["bf16"], 1), "unit": "TFLOP/s",
                         "frac": round(ach / pk["bf16"], 4), "traffic": None,
                         "peak_source": f"measured bf16 burst {pk['bf16']} TF/s ({pk['src']}), fp16 = bf16 rate"},
            "prefill_q1": {"ms": round(ms_a, 4), "tops": round(ops_attn / (ms_a * 1e-3) / 1e12, 1)},
            "config": {"workload": "NEXT-3 fused Q projection + stage-1 Q quantisation (P:660), configs[1] shape "
                                   "(B=8, N=4096, D=4096 -> 32 heads x d=128), then the prefill on the INT8 query",
                       "parallelism": f"{world} rank(s), each its own batch, no collective"}}


def run_decode_long(args, rank, world, device):
    """configs[4]: 128k-context decode, batch 16 (Llama-3-8B attention shape,
    32/8 heads, mixed INT4/INT2), cache sequence-sharded over the ranks; per
    step: append (last rank) + local split-KV decode + all-gather + LSE merge."""
    import torch

    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import parallel, synth

    c = CFG_LONG
    B, N, Hq, Hkv, d = c["B"], c["N"], c["Hq"], c["Hkv"], c["d"]
    t0, t1 = parallel.seq_shard_tokens(N, world, rank)
    n_loc = t1 - t0
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, alpha_mode=1)
    cache = ta.KVCache(B, Hkv, d, max_blocks=n_loc // 64 + 4, bits=bits, device=device)
    _, k, v = synth.qkv_torch(9009 + rank, B, n_loc, Hkv, Hkv, d, device=device)
    if world > 1:  # global universal scale: one all-reduce(MAX) at cache construction (parallel.py)
        parallel.prefill_seq_sharded(p, cache, k, v, torch.distributed.group.WORLD)
    else:
        ta.turbo_quantize_kv(p, cache, k, v)
    del k, v
    torch.cuda.empty_cache()
    last = rank == world - 1
    toks = [tuple(x[:, 0].contiguous() for x in synth.qkv_torch(7000 + i, B, 1, Hq, Hkv, d, device=device))
            for i in range(args.warmup + args.steps)]
    group = torch.distributed.group.WORLD if world > 1 else None
    st = torch.cuda.current_stream()

    def step(i):
        qd, kd, vd = toks[i]
        if last:
            ta.turbo_quantize_kv(p, cache, kd, vd, mode=1)
        if world > 1:
            return parallel.decode_seq_sharded(p, cache, qd, group, n_splits_local=args.decode_splits)
        o, _, L = ta.turbo_attention_decode(p, cache, qd, n_splits=args.decode_splits)
        return o, L

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = Clocks(device) if rank == 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(args.steps):
        step(args.warmup + i)
    e1.record(st)
    torch.cuda.synchronize()
    clocks = clk.stop() if clk else None
    ms = _max_over_ranks(e0.elapsed_time(e1), world, device) / args.steps
    nblk = cache.n_tokens // 64
    byt = decode_bytes(B, Hkv, d, nblk, cache.n_tokens % 64, bits, Hq)
    total = _max_over_ranks(float(byt), world, device) * world  # shards are equal up to one block
    # roofline of the local decode (kernel + in-GPU split combine), timed alone on this rank
    qd0 = toks[-1][0]
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(st)
    for _ in range(args.steps):
        ta.turbo_attention_decode(p, cache, qd0, with_buffer=last, n_splits=args.decode_splits,
                                  want_fp16=world == 1, want_f32=world > 1)
    d1.record(st)
    torch.cuda.synchronize()
    dec_ms = d0.elapsed_time(d1) / args.steps
    pk = peaks()
    roof = {"bound": "hbm", "kernel": "decode_kernel + combine (rank 0)", "achieved": round(byt / (dec_ms * 1e-3) / 1e9, 1),
            "peak": pk["hbm"], "unit": "GB/s", "frac": round(byt / (dec_ms * 1e-3) / 1e9 / pk["hbm"], 4),
            "traffic": None, "peak_source": pk["src"]}
    return {"value": total / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_step": ms, "scaling": "strong",
            "clocks": clocks, "roofline": roof,
            "tokens_per_s": B / (ms * 1e-3),
            "config": {"workload": "configs[4]: decode 128k context, batch 16, Llama-3-8B attention shape "
                                   "(32 Q / 8 KV heads, d=128), mixed INT4/INT2; step = append + split-KV decode "
                                   "+ all-gather + LSE combine",
                       "parallelism": f"sequence-sharded cache over {world} rank(s), NCCL all-gather of (O, L)",
                       "decode_splits_per_rank": args.decode_splits}}


def relaunch_under_torchrun(n):
    """`python bench.py --gpus N` without torchrun: check that N GPUs are visible, then re-execute
    this command as N ranks on this node (torch.distributed.run, 127.0.0.1 rendezvous)."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n:
        sys.exit(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--splits", type=int, default=None,
                    help="split-KV count of the decode in the step (default: auto_splits; 0: balanced)")
    ap.add_argument("--decode-splits", type=int, default=None,
                    help="decode split count (default: binding.auto_splits; 0: the balanced schedule)")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-deviation", action="store_true", help="skip the deviation-from-exact report")
    ap.add_argument("--workload", default="step",
                    choices=["step", "prefill_70b", "decode_long", "prefill_chunk", "q_projection"],
                    help="step = the default hot-path step (configs[1] + configs[2] decode)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        relaunch_under_torchrun(args.gpus)  # one rank per GPU (does not return)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch

    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                 f"(torchrun --nproc-per-node {args.gpus}, or plain `python bench.py --gpus {args.gpus}`)")
    if torch.cuda.device_count() < world or local >= torch.cuda.device_count():
        sys.exit(f"bench.py: {world} rank(s) requested but only {torch.cuda.device_count()} GPU(s) visible")

    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2412_08585_b200 import build

    build.build()
    if args.workload != "step":
        fn = {"prefill_70b": run_prefill_70b, "decode_long": run_decode_long,
              "prefill_chunk": run_prefill_chunk, "q_projection": run_q_projection}[args.workload]
        res = fn(args, rank, world, local)
        if rank == 0:
            line = {"metric": BASE_METRIC, "value": round(res["value"], 2), "unit": res["unit"], "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_step"], 4),
                    "higher_is_better": True, "scaling": res["scaling"], "vs_baseline": None,
                    "dtype": res.get("dtype", "int8"), "data": "synthetic", "config": res["config"]}
            if "tokens_per_s" in res:
                line["tokens_per_s"] = round(res["tokens_per_s"], 1)
            for key in ("clocks", "roofline", "prefill_q1"):
                if key in res:
                    line[key] = res[key]
            print(json.dumps(line), flush=True)
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    res = run_ours(args, rank, world, local)
    cpu = cpu_sample_oracle() if rank == 0 and world == 1 else None
    if rank == 0:
        line = {"metric": BASE_METRIC, "value": round(res["value"], 2), "unit": "TOPS", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_step"], 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
                "data": "synthetic (seeded N(0,1) Q/K/V with outlier channels, DESIGN.md §4)",
                "config": workload_config(args), "roofline": res["roofline"], "cpu_baseline": cpu,
                "e2e": res["e2e"], "gpu_launches": res["launches"], "clocks": res["clocks"],
                "breakdown_ms": res["breakdown_ms"], "quantize_kv": res["quantize_kv"], "decode": res.get("decode"),
                "planner": res["planner"], "deviation": None}
        dev = {}
        if res.get("deviation"):
            dev.update(res["deviation"])
        if line["decode"] and line["decode"].get("deviation"):
            dev["decode_configs2"] = line["decode"].pop("deviation")
        if dev and not args.no_deviation:
            dev["trend_v_probe"] = trend_v_probe(local)
            dev["reference"] = "Eq. 2 (PAPER.md:229-233) in FP64 on the same fp16 inputs"
        line["deviation"] = dev or None
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
