#!/usr/bin/env python
"""Benchmark: BASELINE config 5 -- data-parallel MLP training step, samples/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One step = forward of 4 x Linear(4096,4096)+ReLU + Linear(4096,1000) over the
rank's shard of the 65536-sample global batch, mean cross-entropy, backward,
gradient all-reduce over NCCL (N > 1), one fused Adam(lr=1e-3) update. fp32
everywhere (3xBF16 tcgen05 GEMMs = fp32 accuracy). Global batch fixed ->
strong scaling. Timing: W warm-up steps, barrier + device sync, CUDA events on
the engine stream around exactly K steps, max over ranks. Inputs (1 GiB per
rank at N=1) are larger than L2, so no explicit flush.

Keys beyond the base contract:
  e2e         same metric through the public API with the batch copied
              host(pinned)->device every step and the loss read back
  roofline    dominant kernel (tcgen05 3xBF16 GEMM): algorithmic FLOPs per
              launch / its CUDA-event duration inside a real step
  cpu_baseline  the NumPy oracle port of the reference on this host's cores
  ops         the per-op benchmarks of configs 2-4 (1 GPU, rank 0)
"""

from __future__ import annotations

import argparse
import collections
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

GLOBAL_BATCH = 65536
WIDTH, CLASSES, DEPTH = 4096, 1000, 4
METRIC = "MLP train samples/s (BASELINE config 5: 4x4096 + 4096->1000, global batch 65536, Adam)"


def flops_per_step(batch):
    """fwd 2*B*(4*4096^2 + 4096*1000); dW same; dX for layers 2..5 (x needs no grad)."""
    fw = 2 * batch * (DEPTH * WIDTH * WIDTH + WIDTH * CLASSES)
    dx = 2 * batch * ((DEPTH - 1) * WIDTH * WIDTH + WIDTH * CLASSES)
    return fw + fw + dx


# --------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.time(), parts))

    def window(self, t0, t1):
        """Keep only the samples taken inside [t0, t1] (the timed region). The
        sampler is started before the warm-up: nvidia-smi's start-up (NVML
        init) can stall the CUDA process's launches for hundreds of ms, which
        must not land in a timed step."""
        self.t0, self.t1 = t0, t1

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        lo, hi = getattr(self, "t0", 0.0), getattr(self, "t1", float("inf"))
        self.rows = [r for t, r in self.rows if lo <= t <= hi]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def ncu_traffic():
    """dram bytes per launch of the GEMM kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("flops_per_launch")
    except Exception:
        return None, None


# --------------------------------------------------------------------- reference arm


class CpuSampleStep:
    """One bounded sample of the config-5 step on the host cores through the
    NumPy f64 restatement of the reference (oracle/tensorlite_np.py): the
    step's work cut into GLOBAL_BATCH / rows equal slices and one slice timed
    -- forward + backward over `rows` samples (every FLOP of the step scales
    with the batch rows) plus the Adam update of the same 1/(GLOBAL_BATCH/rows)
    share of every parameter tensor (its rows). value = rows / seconds, the
    same samples/s as the device arm; nothing is extrapolated from a fit."""

    def __init__(self, rows=1024, seed=0):
        from oracle import tensorlite_np as O
        from paper_2602_00125_b200.data import mlp_config5

        self.O = O
        self.rows = rows
        self.params = mlp_config5(seed, WIDTH, CLASSES, DEPTH)
        rng = np.random.default_rng(1)
        self.x = rng.standard_normal((rows, WIDTH), dtype=np.float32)
        self.labels = rng.integers(0, CLASSES, rows)
        self.frac = rows / GLOBAL_BATCH
        self.adam = O.Adam(lr=1e-3)

        class _NoOpt:
            def step(self, key, th, g):
                return th

        self._noopt = _NoOpt()

    def run(self):
        O = self.O
        t0 = time.perf_counter()
        r = O.mlp_train_step(self.params, self.x, self.labels, self._noopt)
        for i, ((w, b), (gw, gb)) in enumerate(zip(self.params, r["grads"])):
            kw = max(1, int(round(w.shape[0] * self.frac)))
            kb = max(1, int(round(b.shape[0] * self.frac)))
            self.adam.step(("w", i), w[:kw], gw[:kw])
            self.adam.step(("b", i), b[:kb], gb[:kb])
        return time.perf_counter() - t0

    def describe(self):
        return (f"1/{GLOBAL_BATCH // self.rows} of a config-5 step per timed step: fwd+bwd over "
                f"{self.rows} of the 65536 rows + Adam over the same share of every parameter "
                f"tensor (oracle/tensorlite_np.py, NumPy f64 BLAS on {os.cpu_count()} threads)")


def cpu_oracle_step_rate(rows=1024, reps=3):
    """The CPU baseline of the device arm: median of `reps` timed sample steps."""
    st = CpuSampleStep(rows)
    st.run()  # warm-up (BLAS threads, page-in)
    ts = [st.run() for _ in range(reps)]
    return rows / statistics.median(ts), st.describe()


def run_reference(args):
    """The reference arm: the reference's CPU path (its NumPy restatement;
    the pure-Python reference cannot travel to the GPU box) on all host
    cores, K timed steps of a bounded 1/64 sample of the config-5 workload.
    Under torchrun rank 0 alone runs and prints."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    st = CpuSampleStep()
    for _ in range(max(args.warmup, 0)):
        st.run()
    ts = [st.run() for _ in range(args.steps)]
    v = st.rows * len(ts) / sum(ts)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(ts) / len(ts) * 1000.0, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (fp32 stores)",
        "data": "synthetic (seeded N(0,1) inputs, uniform labels; reference Dense init)",
        "config": {"workload": f"config5_mlp_4x4096_1000_b{GLOBAL_BATCH}_adam",
                   "global_batch": GLOBAL_BATCH, "sample_rows_per_step": st.rows,
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port",
                         "sample": st.describe()},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_ops_baseline():
    """The per-op figures of `op_benchmarks` for the NumPy oracle port on the
    host cores (configs 1, 2 and 3 at 1024 at full size), same
    units: GB/s of algorithmic bytes, TFLOP/s, us/step."""
    from oracle import tensorlite_np as O

    def best(fn, reps=3):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    out = {"kind": "port", "cores": os.cpu_count(), "note": "oracle/tensorlite_np.py (f64 NumPy), best of 3"}
    rng = np.random.default_rng(0)
    a = rng.standard_normal((4096, 4096), dtype=np.float32)
    b = rng.uniform(-1, 1, (1, 4096)).astype(np.float32)
    n = a.size
    out["config2_fused_fwd_gbs"] = 8 * n / best(lambda: O.relu(O.add(O.mul(a, b), b))) / 1e9
    out["config2_exp_gbs"] = 8 * n / best(lambda: O.exp(a)) / 1e9
    out["config2_mul_bcast_gbs"] = 8 * n / best(lambda: O.mul(a, b)) / 1e9
    for ax in (0, 1):
        out[f"config2_sum_dim{ax}_gbs"] = 4 * n / best(lambda: O.axis_sum(a, ax)) / 1e9
        out[f"config2_max_dim{ax}_gbs"] = 4 * n / best(lambda: O.axis_max(a, ax)) / 1e9
    out["config2_sum_all_gbs"] = 4 * n / best(lambda: O.axis_sum(a, None)) / 1e9
    A = rng.uniform(-1, 1, (1024, 1024)).astype(np.float32)
    B = rng.uniform(-1, 1, (1024, 1024)).astype(np.float32)
    dC = rng.standard_normal((1024, 1024), dtype=np.float32)
    out["config3_n1024_fwdbwd_tflops"] = 6 * 1024 ** 3 / best(lambda: O.matmul_fwd_bwd(A, B, dC)) / 1e12
    from paper_2602_00125_b200.data import linear_params

    r1 = np.random.default_rng(0)
    params = [linear_params(r1, 784, 256), linear_params(r1, 256, 10)]
    x1 = r1.standard_normal((256, 784), dtype=np.float32)
    l1 = r1.integers(0, 10, 256)
    out["config1_us_per_step"] = best(lambda: O.mlp_train_step(params, x1, l1, O.SGD(lr=0.01))) * 1e6
    return out


# --------------------------------------------------------------------- op benchmarks (configs 2-4)


def op_benchmarks():
    import paper_2602_00125_b200 as P
    from paper_2602_00125_b200 import _lib as L

    out = {}
    from paper_2602_00125_b200 import graph

    def timed(fn, iters):
        """Device time per call: `iters` calls captured into one CUDA graph and
        replayed (no Python launch overhead between the kernels)."""
        def body():
            for _ in range(iters):
                fn()

        g = graph.capture(body, warmup=1)
        g.replay()
        L.synchronize()
        e0, e1 = L.Event(), L.Event()
        e0.record()
        g.replay()
        e1.record()
        return e0.elapsed_ms(e1) / iters

    def timed_eager(fn, iters):
        fn()
        L.synchronize()
        e0, e1 = L.Event(), L.Event()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        return e0.elapsed_ms(e1) / iters

    # config 2: fused relu(a*b+b) fwd + fused bwd, and the 6 axis reductions.
    # `a` is 64 MiB (< the 126 MB L2), so the timed loop rotates through 6
    # independent copies (384 MiB) -- every call streams its input from HBM.
    rng = np.random.default_rng(0)
    a0 = rng.standard_normal((4096, 4096), dtype=np.float32)
    copies = [P.from_numpy(a0) for _ in range(6)]
    b = P.from_numpy(rng.uniform(-1, 1, (1, 4096)).astype(np.float32))
    n = 4096 * 4096
    rot = [0]

    def nxt():
        rot[0] = (rot[0] + 1) % len(copies)
        return copies[rot[0]]

    with P.no_grad():
        ms = timed(lambda: P.fused_muladd_relu(nxt(), b), 24)
        out["config2_fused_fwd_gbs"] = 2 * 4 * n / ms / 1e6
        ms = timed(lambda: P.muladd_relu_sum_grads(nxt(), b), 24)
        out["config2_fused_bwd_gbs"] = 2 * 4 * n / ms / 1e6
        ms = timed(lambda: P.exp(nxt()), 24)
        out["config2_exp_gbs"] = 2 * 4 * n / ms / 1e6
        ms = timed(lambda: P.mul(nxt(), b), 24)
        out["config2_mul_bcast_gbs"] = 2 * 4 * n / ms / 1e6
        for ax in (0, 1):
            ms = timed(lambda: P.sum(nxt(), axis=ax), 24)
            out[f"config2_sum_dim{ax}_gbs"] = 4 * n / ms / 1e6
            ms = timed(lambda: P.max(nxt(), axis=ax), 24)
            out[f"config2_max_dim{ax}_gbs"] = 4 * n / ms / 1e6
        ms = timed(lambda: P.sum(nxt()), 24)
        out["config2_sum_all_gbs"] = 4 * n / ms / 1e6
    # the whole config-2 workload as one sequence (what a user runs): relu(a*b+b),
    # exp(clamp(a)), sum/mean/max over dim 0 and dim 1, the full sum, and the
    # gradients of sum(y) w.r.t. a and b (fused op+grad kernel) -- one CUDA graph
    def c2_all():
        a = nxt()
        with P.no_grad():
            y = P.fused_muladd_relu(a, b)
            P.exp(P.clamp(a, -10.0, 10.0))
            for ax in (0, 1):
                P.sum(y, axis=ax)
                P.mean(y, axis=ax)
                P.max(y, axis=ax)
            P.sum(y)
            P.muladd_relu_sum_grads(a, b)

    ms = timed(c2_all, 12)
    out["config2_e2e_us"] = ms * 1000
    # the same workload with ONE read of a (multi-output fusion, bit-identical)
    ms1 = timed(lambda: P.muladd_relu_stats(nxt(), b), 12)
    out["config2_single_pass_us"] = ms1 * 1000
    out["config2_single_pass_gbs"] = 4 * 4 * n / ms1 / 1e6
    # single-pass lower bound: read a once; write y, e, a_bar
    out["config2_e2e_gbs_vs_single_pass_bytes"] = 4 * 4 * n / ms / 1e6
    out["config2_note"] = ("device time per op from a CUDA-graph replay of 24 calls rotating "
                           "over 6 input copies (384 MiB > L2); GB/s = algorithmic bytes "
                           "(read a [+ write out]) / time; roofline_fractions divide by MEASURED_PEAKS.json hbm_gbs")
    del copies, b
    # config 3: square matmul fwd+bwd (3 GEMMs, 6 n^3 flops)
    for size in (1024, 4096, 8192):
        A = P.from_numpy(rng.uniform(-1, 1, (size, size)).astype(np.float32), requires_grad=True)
        B = P.from_numpy(rng.uniform(-1, 1, (size, size)).astype(np.float32), requires_grad=True)
        dC = P.from_numpy(rng.standard_normal((size, size), dtype=np.float32))

        def fb():
            P.reset_tape()
            A.buffer.version += 1  # fresh operands every iteration: no split reuse
            B.buffer.version += 1
            C = P.mm(A, B)
            P.backward(C, seed=dC)

        ms = timed(fb, 3 if size == 8192 else 5)
        out[f"config3_n{size}_fwdbwd_tflops"] = 6 * size ** 3 / ms / 1e9
        if size == 4096:
            # the same three GEMMs on the FP32 pipe (FFMA2, exact fp32 accumulate): the
            # north star's "FP32 SIMT" scheme, against the chip's FP32 peak
            P.set_gemm_algo("simt")
            try:
                ms = timed(fb, 3)
                out["config3_n4096_fwdbwd_fp32_simt_tflops"] = 6 * size ** 3 / ms / 1e9
            except Exception as e:  # noqa: BLE001 -- a secondary figure never costs the others
                out["config3_n4096_fwdbwd_fp32_simt_error"] = f"{type(e).__name__}: {e}"[:200]
            finally:
                P.set_gemm_algo(None)
        del A, B, dC
    P.reset_tape()
    # config 4: softmax(X@W + b), loss = mean(Y*T), full backward
    X = P.from_numpy(rng.standard_normal((64, 512, 1024), dtype=np.float32), requires_grad=True)
    W = P.from_numpy(rng.normal(0, 0.03, (1024, 1024)).astype(np.float32), requires_grad=True)
    bias = P.zeros((1024,), requires_grad=True)
    Tt = P.from_numpy(rng.uniform(0, 1, (64, 512, 1024)).astype(np.float32))

    def c4():
        P.reset_tape()
        X.buffer.version += 1
        W.buffer.version += 1
        Y = P.softmax(P.add(P.mm(X, W), bias))
        P.backward(P.mean(P.mul(Y, Tt)))

    ms = timed(c4, 5)
    out["config4_ms_per_step"] = ms
    out["config4_gemm_tflops_effective"] = 3 * 2 * 32768 * 1024 * 1024 / ms / 1e9
    # the same step written with the fused Linear layer: X @ W + b as one GEMM
    # whose epilogue adds the bias (bit-identical to the separate add)
    X2 = P.reshape(X, (-1, 1024))

    def c4_fused():
        P.reset_tape()
        X.buffer.version += 1
        W.buffer.version += 1
        Y = P.softmax(P.linear(X2, P.transpose2d(W), bias))
        P.backward(P.mean(P.mul(Y, P.reshape(Tt, (-1, 1024)))))

    out["config4_fused_linear_ms_per_step"] = timed(c4_fused, 5)
    # the step as a PyTorch user writes it with fused layers: nn.Linear (bias in
    # the GEMM epilogue) + the fused softmax*T mean loss (one row pass each
    # way; the backward emits the dX/dW GEMMs' operand split and the bias
    # gradient) -- bit-identical to the composition above
    T2 = P.reshape(Tt, (-1, 1024))

    def c4_fused_loss():
        P.reset_tape()
        X.buffer.version += 1
        W.buffer.version += 1
        z = P.linear(X2, P.transpose2d(W), bias)
        P.backward(P.softmax_mul_mean(z, T2))

    out["config4_fused_loss_ms_per_step"] = timed(c4_fused_loss, 5)
    P.reset_tape()
    del X, W, bias, Tt

    # config 1: 784-256-10 MLP, one SGD(lr=0.01) step on 256 samples; eager
    # (one Python-driven launch per op) and replayed as one CUDA graph
    from paper_2602_00125_b200 import nn, optim
    from paper_2602_00125_b200.data import build_mlp, linear_params

    r1 = np.random.default_rng(0)
    c1 = build_mlp([linear_params(r1, 784, 256), linear_params(r1, 256, 10)])
    x1 = P.from_numpy(r1.standard_normal((256, 784), dtype=np.float32))
    l1 = nn.labels_buffer(r1.integers(0, 10, 256))
    sgd = optim.SGD(lr=0.01)

    def c1_step():
        P.reset_tape()
        loss = nn.cross_entropy(c1(x1), l1)
        optim.step_all(sgd, c1.parameters(), P.backward(loss))
        return loss

    ms = timed_eager(c1_step, 20)
    out["config1_eager_us_per_step"] = ms * 1000
    g1 = graph.capture(c1_step, warmup=1)
    g1.replay()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    for _ in range(50):
        g1.replay()
    e1.record()
    ms = e0.elapsed_ms(e1) / 50
    out["config1_graph_us_per_step"] = ms * 1000
    out["config1_graph_samples_per_s"] = 256 / (ms / 1000)
    P.reset_tape()
    # roofline fractions: HBM-bound config-2 ops against the measured copy
    # bandwidth; GEMM-bound configs against the 3xBF16 ceiling (bf16 sustained / 3)
    peaks, _ = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6457.0)
    tc = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1422.1)) / 3.0
    frac = {k.replace("_gbs", "_frac_hbm"): v / hbm for k, v in out.items()
            if k.startswith("config2_") and k.endswith("_gbs")}
    out["config4_fused_gemm_tflops_effective"] = 3 * 2 * 32768 * 1024 * 1024 / out["config4_fused_loss_ms_per_step"] / 1e9
    for k in ("config3_n1024_fwdbwd_tflops", "config3_n4096_fwdbwd_tflops",
              "config3_n8192_fwdbwd_tflops", "config4_gemm_tflops_effective",
              "config4_fused_gemm_tflops_effective"):
        frac[k.replace("_tflops", "_frac_3xbf16_ceiling")] = out[k] / tc
    # FP32 FFMA peak: 148 SMs x 128 lanes x 2 flops x the maximum SM clock (1965 MHz)
    if "config3_n4096_fwdbwd_fp32_simt_tflops" in out:
        frac["config3_n4096_fwdbwd_fp32_simt_frac_fp32_peak"] = (
            out["config3_n4096_fwdbwd_fp32_simt_tflops"] / (148 * 128 * 2 * 1.965e-3))
    frac["config2_e2e_frac_hbm_single_pass"] = out["config2_e2e_gbs_vs_single_pass_bytes"] / hbm
    frac["config2_single_pass_frac_hbm"] = out["config2_single_pass_gbs"] / hbm
    out["roofline_fractions"] = frac
    return out


# --------------------------------------------------------------------- main arm


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: one process per GPU, the env
    torchrun would set (RANK, LOCAL_RANK, WORLD_SIZE, MASTER_*), NCCL's
    communicator-init lines on stderr (NCCL_DEBUG=INFO unless set). Rank 0
    prints the JSON line; a failing rank takes the others down and the exit
    code is the first failure's."""
    import signal
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries only rank 0's JSON line
        procs.append(subprocess.Popen([sys.executable] + sys.argv, env=env, start_new_session=True))
    rc = 0
    live = list(procs)
    while live:
        for p in list(live):
            c = p.poll()
            if c is None:
                continue
            live.remove(p)
            if c != 0 and rc == 0:
                rc = c
                for q in live:  # the process groups this launcher created
                    try:
                        os.killpg(q.pid, signal.SIGTERM)
                    except ProcessLookupError:
                        pass
        time.sleep(0.2)
    sys.exit(rc)


def main():
    global GLOBAL_BATCH
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-ops", action="store_true", help="skip the config 2-4 op benchmarks")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--no-bf16", action="store_true", help="skip the bf16-variant measurement")
    ap.add_argument("--global-batch", type=int, default=GLOBAL_BATCH,
                    help="config-5 global batch (default: BASELINE's 65536; other values are "
                         "for the per-GPU-size characterisation in DESIGN 6, not the headline)")
    ap.add_argument("--gemm", default="auto", choices=["auto", "tf32x", "3xbf16", "3xtf32"],
                    help="fp32-accurate GEMM algorithm for the headline run")
    args = ap.parse_args()
    GLOBAL_BATCH = args.global_batch
    if args.impl == "reference":
        return run_reference(args)
    # B2_BENCH_SPAWN=1 takes the launcher path at N = 1 too (tests exercise it)
    if "WORLD_SIZE" not in os.environ and (args.gpus > 1 or os.environ.get("B2_BENCH_SPAWN") == "1"):
        return spawn_ranks(args.gpus)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env} ranks were launched")

    import paper_2602_00125_b200 as P
    from paper_2602_00125_b200 import _lib as L, dist, nn, optim
    from paper_2602_00125_b200 import core as C
    from paper_2602_00125_b200.data import PinnedFeeder, ScalarReader, batch_shard, build_mlp, mlp_config5

    env = dist.env_from_os()
    # B2_FORCE_NCCL=1: a 1-rank NCCL communicator at N = 1 (the N > 1 code path on one GPU)
    comm = dist.Communicator(env, force_nccl=os.environ.get("B2_FORCE_NCCL") == "1")
    world, rank = env.world, env.rank
    lo, hi = dist.shard_rows(GLOBAL_BATCH, rank, world)
    rows = hi - lo

    model = build_mlp(mlp_config5(0, WIDTH, CLASSES, DEPTH))
    params = model.parameters()
    opt = optim.Adam(lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
    x_np, y_np = batch_shard(1234, rank, rows, WIDTH, CLASSES)

    gemm_log = []
    if args.gemm != "auto":
        P.set_gemm_algo(args.gemm)
    g_algo = C.get_gemm_algo()
    if g_algo is None:
        import ctypes

        sel = ctypes.c_int()
        L.check(L.lib().b2_gemm_select(0, 1, rows, WIDTH, WIDTH, WIDTH, WIDTH, ctypes.byref(sel)))
        g_algo = sel.value
    # Input pipeline (both arms of the measurement): every step takes a new
    # batch -- a feeder slot whose version is bumped, so cached operand splits
    # are stale -- and its 3xBF16 split for the first GEMM is made on the
    # feeder's stream, overlapping the previous step. `value`: the batch is
    # resident in HBM (two slots, uploaded once); e2e: it is copied from
    # pinned host memory every step (H2D on the same stream, before the split).
    presplit = "3xbf16" if g_algo == L.GEMM_3XBF16 else None
    feeder = PinnedFeeder(x_np, y_np, presplit=presplit, classes=CLASSES)
    dev_feeder = PinnedFeeder(x_np, y_np, presplit=presplit, resident=True, classes=CLASSES)
    del x_np
    ALGO_INFO = {
        L.GEMM_TF32X: ("k_gemm_tc<TF32X> (tcgen05 kind::tf32 hi*hi + 2x kind::f16 bf16 cross terms)",
                       4.0, "TF32X = 1 tf32 MMA (half the bf16 rate) + 2 bf16 MMAs per fp32 MAC: "
                            "ceiling = bf16/4",
                       "TF32X tcgen05 (tf32 main + bf16 cross terms, fp32 accuracy ~2e-6)"),
        L.GEMM_3XBF16: ("k_gemm_tc<3xBF16> (tcgen05 kind::f16: hi*hi + hi*lo + lo*hi)", 3.0,
                        "3xBF16 = 3 bf16 MMAs per fp32 MAC: ceiling = bf16/3",
                        "3xBF16 tcgen05 (bf16 hi/lo split, 3 MMAs, fp32 accuracy ~4e-6)"),
        L.GEMM_3XTF32: ("k_gemm_tc<3xTF32>", 6.0, "3xTF32 = 3 tf32 MMAs per MAC: ceiling = bf16/6",
                        "3xTF32 tcgen05 (fp32 accuracy ~1e-6)"),
    }
    a_kernel, a_div, a_note, a_desc = ALGO_INFO[g_algo]

    inflight = collections.deque()

    def step(x, labels, read_loss=False):
        # at most 2 steps queued ahead of the device: the host never runs so far
        # ahead that the caching allocator has to grow the pool mid-run (a
        # multi-GB cudaMalloc stalls the host while the device drains)
        if len(inflight) >= 2:
            inflight.popleft().synchronize()
        P.reset_tape()
        logits = model(x)
        loss = nn.cross_entropy(logits, labels, denom=rows)
        # all-reduce + Adam per layer on a side stream as soon as its last
        # gradient is queued: the updates overlap the remaining backward GEMMs
        red = dist.GradReducer(comm, params, optimizer=opt)
        store = P.backward(loss, on_leaf_ready=red.hook)
        red.finish()
        red.step_rest(store)
        ev = L.Event()
        ev.record()
        inflight.append(ev)
        return loss.item() if read_loss else loss

    sampler = ClockSampler(env.local_rank)
    sampler.start()
    for _ in range(max(args.warmup, 0)):
        step(*dev_feeder.next())
    comm.barrier()
    t_wall0 = time.time()
    n0 = L.launch_count()
    e0, e1 = L.Event(), L.Event()
    marks, host_ms, gc_log = [], [], []
    dbg = bool(os.environ.get("B2_BENCH_DEBUG"))
    if dbg:
        import gc

        def _gc_cb(phase, info, _t=[0.0]):
            if phase == "start":
                _t[0] = time.perf_counter()
            else:
                gc_log.append((info.get("generation"), round((time.perf_counter() - _t[0]) * 1e3, 1)))
        gc.callbacks.append(_gc_cb)
    e0.record()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        last = step(*dev_feeder.next())
        if dbg:
            host_ms.append(round((time.perf_counter() - t0) * 1e3, 1))
            ev = L.Event()
            ev.record()
            marks.append(ev)
    e1.record()
    L.synchronize()
    if marks:
        gc.callbacks.remove(_gc_cb)
        prev, per = e0, []
        for ev in marks:
            per.append(round(prev.elapsed_ms(ev), 2))
            prev = ev
        print("per-step ms:", per, "host ms:", host_ms, "gc:", gc_log, "allocator:", L.alloc_stats(),
              file=sys.stderr)
    launches = L.launch_count() - n0
    sampler.window(t_wall0, time.time())
    comm.barrier()
    ms_local = e0.elapsed_ms(e1) / args.steps
    clocks = sampler.stop()
    ms = comm.max_scalar(ms_local)
    value = GLOBAL_BATCH / (ms / 1000.0)
    loss_val = last.item()

    # e2e: same step through the public API, batch H2D from pinned host memory
    # every step and the loss read back to the host every step
    # every step's loss is read back through a pinned slot; step i's value is
    # taken after step i+1 is queued (ScalarReader), so the stream never drains
    reader = ScalarReader()
    for _ in range(2):
        xb, yb = feeder.next()
        reader.read(step(xb, yb))
    reader.flush()
    comm.barrier()
    e2, e3 = L.Event(), L.Event()
    e2.record()
    e2e_losses = []
    for _ in range(args.steps):
        xb, yb = feeder.next()
        v = reader.read(step(xb, yb))
        if v is not None:
            e2e_losses.append(v)
    e2e_losses.append(reader.flush())
    e3.record()
    L.synchronize()
    assert len(e2e_losses) == args.steps and all(np.isfinite(e2e_losses))
    comm.barrier()
    ms_e2e = comm.max_scalar(e2.elapsed_ms(e3) / args.steps)

    # roofline of the dominant kernel: time every GEMM launch of one step
    # (3 steps; the share is against the same 3 steps' device time)
    t_steps = 3
    C.GEMM_TIMER = gemm_log
    e4, e5 = L.Event(), L.Event()
    e4.record()
    for _ in range(t_steps):
        step(*dev_feeder.next())
    e5.record()
    L.synchronize()
    C.GEMM_TIMER = None
    timed_step_ms = e4.elapsed_ms(e5) / t_steps
    g_flops = sum(f for f, _, _ in gemm_log) / t_steps
    g_ms = sum(s.elapsed_ms(e) for _, s, e in gemm_log) / t_steps
    n_gemm = len(gemm_log) // t_steps
    achieved = g_flops / (g_ms / 1000.0) / 1e12
    peaks, src = measured_peaks()
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    traffic, tr_flops = ncu_traffic()
    # an fp32-accurate tensor-core scheme is bounded by its own
    # ceiling -- the measured bf16 dense peak / the bf16-equivalent MMAs it
    # spends per fp32 MAC (3xBF16: 3) -- in fp32-equivalent (algorithmic) flops
    ceiling = peak / a_div
    roof = {
        "bound": "tensor", "achieved": achieved, "peak": ceiling,
        "unit": "TFLOP/s (fp32-equivalent)", "frac": achieved / ceiling, "traffic": traffic,
        "kernel": a_kernel,
        "algorithmic_flops_per_step": g_flops, "gemm_launches_per_step": n_gemm,
        "gemm_ms_per_step": g_ms, "gemm_share_of_step": g_ms / timed_step_ms,
        "peak_source": f"{src} bf16 dense sustained (MEASURED_PEAKS.json) {peak} / {a_div:g}",
        "bf16_peak": peak, "frac_of_bf16_peak": achieved / peak,
        "note": a_note,
    }

    def variant(algo, desc, kernel, div):
        """The same step with another GEMM scheme: K timed steps after warm-up
        (the variant's casts/splits allocate new blocks: two extra warm-up
        steps let the pool settle) + 3 steps with every GEMM launch timed."""
        P.set_gemm_algo(algo)
        sp_saved, dev_feeder.sp = dev_feeder.sp, None  # the variant splits/casts x itself
        try:
            for _ in range(max(args.warmup, 3) + 2):
                step(*dev_feeder.next())
            comm.barrier()
            b0, b1 = L.Event(), L.Event()
            b0.record()
            for _ in range(args.steps):
                lb = step(*dev_feeder.next())
            b1.record()
            L.synchronize()
            comm.barrier()
            ms_b = comm.max_scalar(b0.elapsed_ms(b1) / args.steps)
            blog = []
            C.GEMM_TIMER = blog
            b2, b3 = L.Event(), L.Event()
            b2.record()
            for _ in range(t_steps):
                step(*dev_feeder.next())
            b3.record()
            L.synchronize()
            C.GEMM_TIMER = None
            bt_ms = b2.elapsed_ms(b3) / t_steps
        finally:
            P.set_gemm_algo(None if args.gemm == "auto" else args.gemm)
            dev_feeder.sp = sp_saved
        bf_flops = sum(f for f, _, _ in blog) / t_steps
        bf_ms = sum(s.elapsed_ms(e) for _, s, e in blog) / t_steps
        bf_ach = bf_flops / (bf_ms / 1000.0) / 1e12
        ceil = peak / div
        return {"value": GLOBAL_BATCH / (ms_b / 1000.0), "unit": "samples/s", "ms_per_step": ms_b,
                "dtype": desc, "final_loss": lb.item(),
                "roofline": {"bound": "tensor", "achieved": bf_ach, "peak": ceil,
                             "unit": "TFLOP/s" + ("" if div == 1 else " (fp32-equivalent)"),
                             "frac": bf_ach / ceil, "kernel": kernel,
                             "gemm_ms_per_step": bf_ms, "gemm_share_of_step": bf_ms / bt_ms}}

    # BASELINE's bf16 variant of config 5: bf16 GEMM operands (one kind::f16
    # MMA per MAC), fp32 accumulation, fp32 master weights / Adam / loss
    bf16 = None
    if not args.no_bf16:
        try:
            bf16 = variant("bf16", "bf16 GEMM operands, fp32 accumulate/master weights/Adam",
                           "k_gemm_tc<BF16> (tcgen05 kind::f16, cta_group::2, 512-row pair tiles)", 1.0)
        except Exception as e:  # noqa: BLE001
            bf16 = {"error": f"{type(e).__name__}: {e}"[:300]}
    # the north star's sanctioned fp32 scheme (3xTF32 on tcgen05) for the record
    tf32 = None
    if not args.no_bf16 and g_algo != L.GEMM_3XTF32:
        try:
            tf32 = variant("3xtf32", "fp32 (3xTF32 tcgen05: hi*hi + hi*lo + lo*hi tf32 MMAs)",
                           "k_gemm_tc<3xTF32> (tcgen05 kind::tf32)", 6.0)
        except Exception as e:  # noqa: BLE001
            tf32 = {"error": f"{type(e).__name__}: {e}"[:300]}

    ops = None
    cpu = None
    ops_cpu = None
    if rank == 0 and world == 1:
        # the secondary measurements never cost the headline line: a failure is
        # recorded in the JSON instead of ending the run
        if not args.no_ops:
            try:
                ops = op_benchmarks()
            except Exception as e:  # noqa: BLE001
                ops = {"error": f"{type(e).__name__}: {e}"[:300]}
        if not args.no_cpu:
            try:
                v_cpu, desc = cpu_oracle_step_rate()
                cpu = {"value": v_cpu, "unit": "samples/s", "cores": os.cpu_count(), "kind": "port",
                       "sample": desc + "; median of 3 timed sample steps"}
                ops_cpu = cpu_ops_baseline()
            except Exception as e:  # noqa: BLE001
                ops_cpu = {"error": f"{type(e).__name__}: {e}"[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic (seeded N(0,1) inputs, uniform labels; reference Dense init)",
            "config": {"workload": f"config5_mlp_4x4096_1000_b{GLOBAL_BATCH}_adam",
                       "global_batch": GLOBAL_BATCH, "per_gpu_batch": rows,
                       "layers": "4xLinear(4096,4096)+ReLU, Linear(4096,1000)",
                       "optimizer": "Adam lr=1e-3 betas=(0.9,0.999) eps=1e-8",
                       "gemm": a_desc,
                       "parallelism": f"dp{world}", "l2": "inputs > L2 (1 GiB/rank at N=1)",
                       "input_pipeline": "2 batch slots (value: resident in HBM; e2e: H2D from pinned "
                                         "host every step); each step's 3xBF16 split of its batch is made "
                                         "on the feeder stream, overlapping the previous step"},
            "e2e": {"value": GLOBAL_BATCH / (ms_e2e / 1000.0), "unit": "samples/s",
                    "h2d_bytes_per_step": feeder.h2d_bytes, "d2h_bytes_per_step": 4},
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
            "allocator": L.alloc_stats(),
            "launches_per_step": launches / args.steps,
            "tflops_per_gpu": flops_per_step(rows) / (ms / 1000.0) / 1e12,
            "final_loss": loss_val,
            "bf16_variant": bf16,
            "fp32_3xtf32_variant": tf32,
            "ops": ops,
            "ops_cpu_baseline": ops_cpu,
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
