#!/usr/bin/env python3
"""bench.py -- the driver's benchmark contract for the arXiv 2202.08361 hot path.

Default workload (N=1): BASELINE.json configs[1], the batched complex 2x2
Hermitian EVD of r = 2^26 matrices (jsvd_evd2_batched).  One "step" = one
pass of the EVD over the whole batch with inputs resident in HBM (5.1 GB of
algorithmic traffic per step, > L2, so no L2 flush is needed).  Multi-GPU: one
process per GPU (torchrun); the configured batch is split by batch index, rank
k runs matrices [k r/N, (k+1) r/N) (counter-based inputs: shard k == slice k of
the whole batch) -- "scaling": "strong" (the total work is the configured
batch at every N), no data-path collective (the batch shards naturally,
SURVEY 8(e)).  dist_c64 splits configs[4]'s one SVD by column blocks (the
library's NCCL exchange), also strong scaling.

Other workloads (--workload, one JSON line each):
  evd_r64      configs[0]  batched real EVD, r = 2^20 (L2-resident: flushed per step)
  step_r64     configs[2]  one parallel Jacobi sweep step of the 4096 x 1024 real SVD
  gesvj_r64    configs[2]  the full SVD (<= 30 sweeps), sweep-steps/s
  batched_c64  configs[3]  65536 complex 64 x 32 SVDs, SVD/s
  step_c64     configs[4]  one sweep step of the complex 32768 x 8192 SVD (1 GPU)
  dist_c64     configs[4]  jsvd_gesvj sharded by column blocks over the torchrun
                           ranks (NCCL send/recv inside libjsvd), bounded to the
                           first 1024 sweep steps per bench step (one block exchange)

--impl reference: the oracle (oracle/, plain C) on this box's host cores, on a
bounded sample of the same workload per step (this tier's reference arm).
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "2×2 EVDs/s and Jacobi sweep-steps/s; HBM GB/s & % roofline at 1/2/4/8 B200"
FP64_PEAK_INSTR = 148 * 64 * 1.965e9  # FP64 pipe: 64 lanes/clk/SM x 148 SM x 1965 MHz


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_traffic(workload):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# --------------------------------------------------------------- clocks sampler
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML every ~0.2 ms while active
    (the NVML calls release the GIL; the default timed windows are >= ~20 ms)."""

    def __init__(self, dev_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._dev = dev_index
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self._dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "hw_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                "sw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "hw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_power_cap": getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for k, v in names.items():
                            if r & v:
                                self.reasons.add(k)
                    except Exception:
                        pass
                    time.sleep(0.0002)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML unavailable: report nothing rather than guess
            self.error = str(e)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _ncores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# --------------------------------------------------------------- workloads
# workload descriptions shared by both arms (config.workload of the JSON line)
DESC = {
    "evd_c64": "BASELINE configs[1]: batched complex Hermitian 2x2 EVD, fp64, r=2^26 (split over the GPUs), seed 7",
    "evd_r64": "BASELINE configs[0]: batched real symmetric 2x2 EVD, fp64, r=2^20 (split over the GPUs), seed 42",
    "evd_c32": ("single-precision analogue of BASELINE configs[1] (NEXT-1, P:709-717): "
                "batched complex Hermitian 2x2 EVD, fp32, r=2^26 (split over the GPUs), seed 7"),
    "batched_c64": ("BASELINE configs[3]: batch of 65536 complex fp64 64x32 matrices (split over "
                    "the GPUs), re,im ~ N(0,1), full Jacobi SVD (U, Sigma, V) of each, seed 4"),
    "norm_c64": ("NEXT-3 (Alg SM6.3): one-pass (e,f) Frobenius norms of the 8192 columns of "
                 "BASELINE configs[4]'s complex fp64 32768x8192 matrix, s = 32 lanes"),
}


class EvdWorkload:
    """configs[0] / configs[1]: batched 2x2 EVD (jsvd_evd2_batched)."""
    graphable = True

    def __init__(self, name, rank, world):
        import torch
        import synth
        self.name = name
        self.cplx = name in ("evd_c64", "evd_c32")
        self.f32 = name == "evd_c32"
        self.r_total = (1 << 26) if self.cplx else (1 << 20)
        self.r = self.r_total // world  # this rank's shard of the configured batch
        self.unit = "EVD/s"
        off = rank * self.r
        if self.f32:
            self.desc = DESC["evd_c32"]
            self.host = synth.evd_cfg2_f32(self.r, off=off)
        elif self.cplx:
            self.desc = DESC["evd_c64"]
            self.host = synth.evd_cfg2(self.r, off=off)
        else:
            self.desc = DESC["evd_r64"]
            self.host = synth.evd_cfg1(self.r, off=off)
        w = 4 if self.f32 else 8
        self.unit_bytes = (9 * w + 4 + 1 / 8) if self.cplx else (7 * w + 4 + 1 / 8)
        fdt = torch.float32 if self.f32 else torch.float64
        # configs[0] is 63 MB (< 126 MB L2): the steps cycle through separate
        # input/output sets (> 252 MB in all, > L2), so every launch streams from HBM
        self.nsets = 1 if self.cplx else 4 * world
        keys = ("lam1", "lam2", "cos", "sin_re") + (("sin_im",) if self.cplx else ())
        self.sets = []
        for _ in range(self.nsets):
            dev = [torch.from_numpy(a).cuda() for a in self.host]
            out = {k: torch.empty(self.r, dtype=fdt, device="cuda") for k in keys}
            if not self.cplx:
                out["sin_im"] = None
            out["zeta"] = torch.empty(self.r, dtype=torch.int32, device="cuda")
            out["perm"] = torch.empty((self.r + 31) // 32, dtype=torch.int32, device="cuda")
            self.sets.append((dev, out))
        self.dev, self.out = self.sets[0]
        self.k = 0
        self.units_per_step = self.r
        self.kernel = "evd2f_vec4_kernel" if self.f32 else ("evd2_vec2_kernel" if self.cplx else "evd2_scalar_kernel")
        self.l2_note = ("inputs+outputs %.1f GB per step per GPU > 126 MB L2 (no flush needed)"
                        % (self.unit_bytes * self.r / 1e9)) if self.cplx else \
            ("%.0f MB per step per GPU; steps cycle through %d input/output sets (%.0f MB > 126 MB L2)"
             % (self.unit_bytes * self.r / 1e6, self.nsets, self.nsets * self.unit_bytes * self.r / 1e6))

    def prepare(self):
        pass

    def step(self, stream):
        import paper_2202_08361_b200 as J
        dev, out = self.sets[self.k % self.nsets]
        self.k += 1
        J.evd2_batched(*dev, out=out, stream=stream)

    def bytes_per_step(self):
        return self.unit_bytes * self.r

    def e2e(self, stream, steps):
        import torch
        import paper_2202_08361_b200 as J
        # the C-ABI host-buffer entry (jsvd_evd2_batched_host): pinned host
        # inputs/outputs, chunked H2D / kernel / D2H over three internal streams
        hin = [torch.from_numpy(a).pin_memory() for a in self.host]
        if not self.cplx:
            hin.append(None)
        hout = {k: (torch.empty(v.shape, dtype=v.dtype).pin_memory() if v is not None else None)
                for k, v in self.out.items()}
        chunk = min(1 << 21, max(32, (self.r // 8) // 32 * 32))  # >= 8 chunks in flight
        dt = torch.float32 if self.f32 else torch.float64
        work = torch.empty(J.evd2_host_workspace(dt, self.cplx, chunk), dtype=torch.uint8,
                           device="cuda")

        def one():
            J.evd2_batched_host(*hin, out=hout, chunk=chunk, work=work, stream=stream)

        one()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            one()
        e1.record(stream)
        torch.cuda.synchronize()
        self.e2e_note = f"jsvd_evd2_batched_host, pinned host buffers, chunk {chunk}, 3 streams"
        h2d = sum(a.nbytes for a in self.host)
        d2h = sum(v.numel() * v.element_size() for v in self.out.values() if v is not None)
        return e0.elapsed_time(e1), h2d, d2h

    def cpu_sample(self):
        """(seconds per call, units per call, description) of the oracle on a sample."""
        import oracle as O
        n = min(self.r, 1 << 20)
        sl = [a[:n] for a in self.host]
        fn = O.evd2_batched_f32 if self.f32 else O.evd2_batched
        fn(*[a[:1024] for a in sl])
        return lambda: fn(*sl), n, f"the first {n} matrices of the batch per call"


class StepWorkload:
    """configs[2]: one parallel Jacobi step (jsvd_sweep_step) of the 4096 x 1024
    real SVD, steps 0.. of the first sweep (every pair transformed), G and V as
    jsvd_gesvj leaves them after its initial scaling (Eq. skn) and V = I."""
    graphable = True

    def __init__(self, name, rank, world):
        import torch
        import synth
        import paper_2202_08361_b200 as J
        self.name, self.unit = name, "sweep-steps/s"
        self.desc = ("BASELINE configs[2]: real fp64 one-sided Jacobi SVD 4096x1024, "
                     "sigma geometric 1->1e-12, one round-robin sweep step (n/2 = 512 pairs)")
        A, _ = synth.svd_cfg3()
        self.m, self.n = A.shape
        k = int(np.floor(np.log2(np.abs(A).max())))
        s0 = (1022 - int(np.floor(np.log2(self.m)))) - k - 1  # Eq. (skn), as jsvd_gesvj
        self.A0 = np.ldexp(A, s0)
        self.G = torch.from_numpy(np.ascontiguousarray(self.A0.T)).cuda().T
        self.V = torch.eye(self.n, dtype=torch.float64, device="cuda").T  # column-major view
        self.pairs = torch.empty((self.n - 1, self.n), dtype=torch.int32, device="cuda")
        for s in range(self.n - 1):
            J.strategy_pairs(self.n, self.n, s, out=self.pairs[s])
        self.ce = torch.empty(self.n, dtype=torch.float64, device="cuda")
        self.cf = torch.empty(self.n, dtype=torch.float64, device="cuda")
        self.t = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.mm = torch.zeros(1, dtype=torch.float64, device="cuda")
        self.k = 0
        self.units_per_step = 1
        self.kernel = "step_kernel<0,256,1,16>"
        self.l2_note = "G (32 MB) + V (8 MB) are L2-resident across steps, as in the real iteration"

    def prepare(self):
        pass

    def reset_counters(self):
        self.t.zero_()

    def step(self, stream):
        import paper_2202_08361_b200 as J
        J.sweep_step(self.G, self.V, self.pairs[self.k % (self.n - 1)], col_e=self.ce,
                     col_f=self.cf, t_dev=self.t, mmax_dev=self.mm, stream=stream)
        self.k += 1

    def bytes_for(self, steps, transformed):
        w = 8
        npairs = self.n // 2
        skipped = npairs * steps - transformed
        return transformed * (4 * self.m * w + 4 * self.n * w) + skipped * 2 * self.m * w

    def e2e(self, stream, steps):
        import torch
        import paper_2202_08361_b200 as J
        hA = torch.from_numpy(np.ascontiguousarray(self.A0.T)).pin_memory()
        hG = torch.empty_like(hA).pin_memory()
        hV = torch.empty((self.n, self.n), dtype=torch.float64).pin_memory()
        Gt = torch.empty((self.n, self.m), dtype=torch.float64, device="cuda")
        V = torch.eye(self.n, dtype=torch.float64, device="cuda").T
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(steps):
            Gt.copy_(hA, non_blocking=True)
            J.sweep_step(Gt.T, V, self.pairs[s], col_e=self.ce, col_f=self.cf, t_dev=self.t,
                         mmax_dev=self.mm, stream=stream)
            hG.copy_(Gt, non_blocking=True)
            hV.copy_(V, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), hA.numel() * 8, (hG.numel() + hV.numel()) * 8

    def cpu_sample(self):
        import oracle as O
        import paper_2202_08361_b200 as J
        W, c, offs = J.step_rspec(False, self.m)
        R = O.RSpec.make(W, c, offs)
        G = np.asfortranarray(self.A0.copy())
        V = np.asfortranarray(np.eye(self.n))
        pairs = O.strategy_pairs(self.n, self.n, 0)
        return lambda: O.step(G, V, pairs, R), 1, "one full step (512 pairs, 4096 x 1024) per call"


class BatchedWorkload:
    """configs[3]: 65536 independent complex 64 x 32 SVDs (jsvd_gesvj_batched),
    full convergence of every matrix per step."""

    def __init__(self, name, rank, world):
        import torch
        import synth
        self.name, self.unit = name, "SVD/s"
        self.b, self.m, self.n = 65536 // world, 64, 32  # this rank's shard
        self.desc = DESC["batched_c64"]
        self.host = synth.svd_cfg4(self.b, off=rank * self.b)
        self.A0 = torch.from_numpy(np.ascontiguousarray(np.transpose(self.host, (0, 2, 1)))).cuda()
        self.A = torch.empty_like(self.A0)
        self.V = torch.empty((self.b, self.n, self.n), dtype=torch.complex128, device="cuda")
        self.sig = torch.empty((self.b, self.n), dtype=torch.float64, device="cuda")
        self.sw = torch.empty(self.b, dtype=torch.int32, device="cuda")
        self.st = torch.empty(self.b, dtype=torch.int32, device="cuda")
        self.tr = torch.empty(self.b, dtype=torch.int64, device="cuda")
        self.units_per_step = self.b
        self.kernel = "batched_fast_kernel<1,0>"
        self.l2_note = "2.1 GB of input per step > L2; A restored from a pristine copy before each step (untimed)"

    def prepare(self):
        self.A.copy_(self.A0)

    def step(self, stream):
        import paper_2202_08361_b200 as J
        J.gesvj_batched(self.A.transpose(1, 2), V=self.V.transpose(1, 2), sigma=self.sig,
                        sweeps=self.sw, status=self.st, stream=stream, transforms=self.tr)

    def fp64_ops(self):
        """Algorithmic FP64 operations of the last step (div, sqrt = 1):
        per pair-step 16m + 12 (norms, dot, test), per transformed pair-step
        12m + 12n + 60 (rotations of G and V, Grammian, EVD)."""
        m, n = self.m, self.n
        pair_steps = int(self.sw.long().sum().item()) * (n - 1) * (n // 2)
        transformed = int(self.tr.sum().item())
        return pair_steps * (16 * m + 12) + transformed * (12 * m + 12 * n + 60)

    def bytes_per_step(self):
        w = 16
        return self.b * (self.m * self.n * w * 2 + self.n * self.n * w + self.n * 8)

    def e2e(self, stream, steps):
        import torch
        import paper_2202_08361_b200 as J
        # the C-ABI host-buffer entry (jsvd_gesvj_batched_host): pinned host
        # A -> U, V, sigma (+ sweeps, status, transforms), chunked over 3 streams
        hA = self.A0.cpu().pin_memory().transpose(1, 2)
        b, m, n = self.b, self.m, self.n
        hout = dict(U=torch.empty((b, n, m), dtype=torch.complex128).pin_memory().transpose(1, 2),
                    V=torch.empty((b, n, n), dtype=torch.complex128).pin_memory().transpose(1, 2),
                    sigma=torch.empty((b, n), dtype=torch.float64).pin_memory(),
                    sweeps=torch.empty(b, dtype=torch.int32).pin_memory(),
                    status=torch.empty(b, dtype=torch.int32).pin_memory(), transforms=None)
        chunk = 8192
        work = torch.empty(J.gesvj_batched_host_workspace(True, m, n, chunk), dtype=torch.uint8,
                           device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            J.gesvj_batched_host(hA, out=hout, chunk=chunk, work=work, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        self.e2e_note = f"jsvd_gesvj_batched_host, pinned host buffers, chunk {chunk}, 3 streams"
        hU, hV, hs = hout["U"], hout["V"], hout["sigma"]
        return e0.elapsed_time(e1), hA.numel() * 16, (hU.numel() + hV.numel()) * 16 + hs.numel() * 8

    def cpu_sample(self):
        import oracle as O
        import paper_2202_08361_b200 as J
        W, c, offs = J.batched_rspec(True, self.m)
        R = O.RSpec.make(W, c, offs)
        k = 256
        sample = self.host[:k]
        return lambda: O.gesvj_batched(sample, R), k, f"the first {k} matrices of the batch per call"


class GesvjWorkload:
    """configs[2]: the full SVD (jsvd_gesvj, flat round-robin, <= 30 sweeps) of
    the 4096 x 1024 real matrix; one bench step = one whole SVD; the unit is
    the sweep step (n-1 per sweep), so value = sweep-steps/s over the solve."""

    def __init__(self, name, rank, world):
        import torch
        import synth
        import paper_2202_08361_b200 as J
        self.name, self.unit = name, "sweep-steps/s"
        self.desc = ("BASELINE configs[2]: real fp64 one-sided Jacobi SVD of one 4096x1024 "
                     "matrix, sigma geometric 1->1e-12, round-robin, tol sqrt(m) eps, <= 30 sweeps")
        A, self.sig_true = synth.svd_cfg3()
        self.m, self.n = A.shape
        self.host = A
        self.A0 = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
        self.At = torch.empty_like(self.A0)
        self.V = torch.empty((self.n, self.n), dtype=torch.float64, device="cuda")
        self.work = torch.empty(J.gesvj_workspace(False, self.m, self.n), dtype=torch.uint8,
                                device="cuda")
        self.units_per_step = None
        self.kernel = "step_kernel<0,256,1,16>"
        self.l2_note = "G (32 MB) + V (8 MB) L2-resident; A restored before each solve (untimed)"
        self.last = None

    def prepare(self):
        self.At.copy_(self.A0)

    def step(self, stream):
        import paper_2202_08361_b200 as J
        self.last = J.gesvj(self.At.T, max_sweeps=30, V=self.V.T, work=self.work, stream=stream)
        self.units_per_step = self.last["sweeps"] * (self.n - 1)

    def bytes_per_step(self):
        w, T = 8, sum(self.last["tps"])
        steps = self.last["sweeps"] * (self.n - 1)
        return (T * (4 * self.m * w + 4 * self.n * w) + (steps * self.n // 2 - T) * 2 * self.m * w)

    def e2e(self, stream, steps):
        import torch
        import paper_2202_08361_b200 as J
        # the C-ABI host-buffer entry (jsvd_gesvj_host): host A in, host U, V, sigma out
        hA = self.A0.cpu().pin_memory().T  # column-major view of the host matrix
        out = dict(U=torch.empty((self.n, self.m), dtype=torch.float64).pin_memory().T,
                   V=torch.empty((self.n, self.n), dtype=torch.float64).pin_memory().T,
                   sigma=torch.empty(self.n, dtype=torch.float64).pin_memory())
        work = torch.empty(J.gesvj_host_workspace(False, self.m, self.n), dtype=torch.uint8,
                           device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            J.gesvj_host(hA, max_sweeps=30, out=out, work=work, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        self.e2e_note = "jsvd_gesvj_host, pinned host buffers (upload, SVD, download)"
        return e0.elapsed_time(e1), hA.numel() * 8, (self.m * self.n + self.n * self.n + self.n) * 8

    def cpu_sample(self):
        import oracle as O
        import paper_2202_08361_b200 as J
        W, c, offs = J.step_rspec(False, self.m)
        R = O.RSpec.make(W, c, offs)
        s0 = (1022 - int(np.floor(np.log2(self.m)))) - int(np.floor(np.log2(np.abs(self.host).max()))) - 1
        G = np.asfortranarray(np.ldexp(self.host, s0))
        V = np.asfortranarray(np.eye(self.n))
        pairs = O.strategy_pairs(self.n, self.n, 0)
        return lambda: O.step(G, V, pairs, R), 1, "one full sweep step (512 pairs) per call"


class StepC64Workload(StepWorkload):
    """configs[4]: one parallel Jacobi step of the complex 32768 x 8192 SVD
    (4096 pairs, one 8-CTA cluster per pair), block round-robin B = 16 -- the
    ordering of the column-block-sharded run -- first sweep (all pairs
    transformed); G (4.3 GB) + V (1.1 GB) far exceed L2."""

    def __init__(self, name, rank, world):
        import torch
        import synth
        import paper_2202_08361_b200 as J
        self.name, self.unit = name, "sweep-steps/s"
        self.desc = ("BASELINE configs[4]: complex fp64 Jacobi SVD of one 32768x8192 matrix, "
                     "sigma log-uniform [1e-8,1], one block-round-robin (B=16) sweep step, 1 GPU")
        G, _ = synth.svd_cfg5_torch()
        self.m, self.n = G.shape
        mx = torch.view_as_real(G).abs().max().item()
        k = int(np.floor(np.log2(mx)))
        lg = int(np.floor(np.log2(self.m)))
        Fm = 1021 - lg - (1 if self.m * self.m >= 2 ** (2 * lg + 1) else 0)
        s0 = Fm - k - 1  # Eq. (skn), complex
        torch.view_as_real(G).mul_(2.0 ** s0)
        self.G = G
        self.V = torch.eye(self.n, dtype=torch.complex128, device="cuda").T
        self.B = 16
        self.pairs = torch.empty((self.n - 1, self.n), dtype=torch.int32, device="cuda")
        for s in range(self.n - 1):
            J.strategy_pairs(self.n, self.B, s, out=self.pairs[s])
        self.ce = torch.empty(self.n, dtype=torch.float64, device="cuda")
        self.cf = torch.empty(self.n, dtype=torch.float64, device="cuda")
        self.t = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.mm = torch.zeros(1, dtype=torch.float64, device="cuda")
        self.k = 0
        self.units_per_step = 1
        self.kernel = "step_kernel<1,256,8,4,12>"
        self.l2_note = "G 4.3 GB + V 1.1 GB >> L2"

    def bytes_for(self, steps, transformed):
        w = 16
        npairs = self.n // 2
        skipped = npairs * steps - transformed
        return transformed * (4 * self.m * w + 4 * self.n * w) + skipped * 2 * self.m * w

    def e2e(self, stream, steps):
        import torch
        import paper_2202_08361_b200 as J
        hG = torch.empty((self.n, self.m), dtype=torch.complex128).pin_memory()
        hG.copy_(self.G.T)
        hV = torch.empty((self.n, self.n), dtype=torch.complex128).pin_memory()
        Gt = torch.empty((self.n, self.m), dtype=torch.complex128, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(steps):
            Gt.copy_(hG, non_blocking=True)
            J.sweep_step(Gt.T, self.V, self.pairs[s], col_e=self.ce, col_f=self.cf, t_dev=self.t,
                         mmax_dev=self.mm, stream=stream)
            hG.copy_(Gt, non_blocking=True)
            hV.copy_(self.V.T, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), hG.numel() * 16, (hG.numel() + hV.numel()) * 16

    def cpu_sample(self):
        import oracle as O
        import paper_2202_08361_b200 as J
        W, c, offs = J.step_rspec(True, self.m)
        R = O.RSpec.make(W, c, offs)
        npairs = 16  # a bounded sample: 16 of the 4096 pairs of a step
        cols = self.pairs[0][: 2 * npairs].cpu().numpy()
        G = np.asfortranarray(self.G[:, cols.tolist()].cpu().numpy())
        V = np.asfortranarray(np.eye(2 * npairs, dtype=np.complex128))
        pairs = np.arange(2 * npairs, dtype=np.int32).reshape(-1, 2)
        frac = npairs / (self.n // 2)
        return (lambda: O.step(G, V, pairs, R)), frac, \
            f"{npairs} of the {self.n // 2} pairs of a step per call (units = fraction of a step)"


class DistC64Workload:
    """configs[4] sharded by column blocks over the torchrun ranks (N = 1, 2, 4,
    8): jsvd_gesvj with a jsvd_dist (the library's own NCCL communicator,
    bootstrapped over the torch.distributed group; N = 1: a one-rank NCCL
    world, block moves as device copies).  One bench step = one jsvd_gesvj call
    bounded to the first 2b = 1024 sweep steps (opts.max_steps): phase I (511
    steps, no exchange), the first phase-II round (512 steps) with its block
    exchange, and the first step of the next round; the local columns are
    restored from a pristine copy before each call (untimed).  The unit is the
    global sweep step (4096 pairs over all ranks)."""

    def __init__(self, name, rank, world):
        import torch
        import synth
        from paper_2202_08361_b200.dist import NcclDist, local_columns
        self.name, self.unit = name, "sweep-steps/s"
        self.desc = ("BASELINE configs[4]: complex fp64 Jacobi SVD of one 32768x8192 matrix, "
                     f"column blocks (B=16) sharded over {world} GPU(s), "
                     + ("NCCL block exchange inside libjsvd" if world > 1 else
                        "one NCCL rank (block moves as device copies)")
                     + ", the first 1024 sweep steps per call")
        A, _ = synth.svd_cfg5_torch()
        self.m, self.n = A.shape
        self.B = 16
        cols = torch.from_numpy(local_columns(self.n, self.B, rank, world)).cuda()
        self.A0 = A.T[cols].contiguous()  # (n/N, m): the local columns, column-major
        del A
        torch.cuda.empty_cache()
        self.At = torch.empty_like(self.A0)
        self.V = torch.empty((self.A0.shape[0], self.n), dtype=torch.complex128, device="cuda")
        self.nd = NcclDist() if world > 1 else NcclDist.single(flags=0)
        import paper_2202_08361_b200 as J
        self.work = torch.empty(J.gesvj_workspace(True, self.m, self.n, self.B, self.nd.dist),
                                dtype=torch.uint8, device="cuda")
        self.max_steps = 2 * (self.n // self.B)
        self.world = world
        self.units_per_step = self.max_steps / world  # value = world * units * K / t = global steps/s
        self.kernel = "step_kernel<1,256,8,4,12>"
        self.l2_note = "local G + V >> L2; local columns restored before each call (untimed)"
        self.last = None

    def prepare(self):
        self.At.copy_(self.A0)

    def step(self, stream):
        import paper_2202_08361_b200 as J
        self.last = J.gesvj(self.At.T, nblocks=self.B, max_sweeps=1, V=self.V.T, work=self.work,
                            stream=stream, dist=self.nd.dist, n=self.n, max_steps=self.max_steps)

    def bytes_per_step(self):
        """per-GPU algorithmic bytes of one call: every pair of the first sweep
        transforms (read + write G pair, read + write V pair)."""
        w = 16
        pairs = self.max_steps * (self.n // 2) // self.world
        return pairs * (4 * self.m * w + 4 * self.n * w)

    def e2e(self, stream, steps):
        """local columns in from pinned host memory, one bounded call, local U
        (iterate) and V back out."""
        import torch
        import paper_2202_08361_b200 as J
        hA = self.A0.cpu().pin_memory()
        hV = torch.empty(self.V.shape, dtype=self.V.dtype).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            self.At.copy_(hA, non_blocking=True)
            J.gesvj(self.At.T, nblocks=self.B, max_sweeps=1, V=self.V.T, work=self.work,
                    stream=stream, dist=self.nd.dist, n=self.n, max_steps=self.max_steps)
            hA.copy_(self.At, non_blocking=True)
            hV.copy_(self.V, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        self.e2e_note = "jsvd_gesvj (sharded, max_steps 1024) between pinned host copies of the local columns"
        return e0.elapsed_time(e1), hA.numel() * 16, (hA.numel() + hV.numel()) * 16

    def cpu_sample(self):
        import oracle as O
        R = O.RSpec.make(2048, 1, [16, 8, 4, 2, 1, 128, 64, 32, 1024, 512, 256])  # R#15, m = 32768
        npairs = 16
        G = np.asfortranarray(self.A0[: 2 * npairs].cpu().numpy().T)
        V = np.asfortranarray(np.eye(2 * npairs, dtype=np.complex128))
        pairs = np.arange(2 * npairs, dtype=np.int32).reshape(-1, 2)
        return (lambda: O.step(G, V, pairs, R)), npairs / (self.n // 2), \
            f"{npairs} of the {self.n // 2} pairs of a step per call (units = fraction of a step)"


class NormWorkload:
    """NEXT-3: the one-pass (e, f) norms (Alg SM6.3, jsvd_norm_ef) of all 8192
    columns of configs[4]'s complex 32768 x 8192 matrix (4.3 GB, read once)."""
    graphable = True

    def __init__(self, name, rank, world):
        import torch
        import synth
        self.name, self.unit = name, "columns/s"
        self.desc = DESC["norm_c64"]
        G, _ = synth.svd_cfg5_torch()
        self.G = G
        self.m, self.n = G.shape
        self.ce = torch.empty(self.n, dtype=torch.float64, device="cuda")
        self.cf = torch.empty(self.n, dtype=torch.float64, device="cuda")
        self.units_per_step = self.n
        self.kernel = "norm_ef_kernel<1>"
        self.l2_note = "G 4.3 GB >> L2"

    def prepare(self):
        pass

    def step(self, stream):
        import paper_2202_08361_b200 as J
        J.norm_ef(self.G, col_e=self.ce, col_f=self.cf, stream=stream)

    def bytes_per_step(self):
        return self.m * self.n * 16 + self.n * 16

    def e2e(self, stream, steps):
        import torch
        import paper_2202_08361_b200 as J
        hG = torch.empty((self.n, self.m), dtype=torch.complex128).pin_memory()
        hG.copy_(self.G.T)
        he = torch.empty(self.n, dtype=torch.float64).pin_memory()
        hf = torch.empty(self.n, dtype=torch.float64).pin_memory()
        Gt = torch.empty((self.n, self.m), dtype=torch.complex128, device="cuda")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                Gt.copy_(hG, non_blocking=True)
                J.norm_ef(Gt.T, col_e=self.ce, col_f=self.cf, stream=stream)
                he.copy_(self.ce, non_blocking=True)
                hf.copy_(self.cf, non_blocking=True)
            e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), hG.numel() * 16, 2 * self.n * 8

    def cpu_sample(self):
        import oracle as O
        k = 16
        cols = self.G[:, :k].cpu().numpy()
        return lambda: O.norm_ef_cols(cols), k, f"the first {k} columns per call"


class GsWorkload:
    """NEXT-4: the real Gram-Schmidt orthogonalization (Alg SM8.1, jsvd_dgsscl)
    of all 4096 disjoint column pairs of a real 32768 x 8192 matrix (2.1 GB)."""
    graphable = True

    def __init__(self, name, rank, world):
        import torch
        import paper_2202_08361_b200 as J
        self.name, self.unit = name, "pairs/s"
        self.desc = ("NEXT-4 (Alg SM8.1): Gram-Schmidt of g_q against g_p for the 4096 pairs of a real "
                     "fp64 32768x8192 matrix (configs[4]'s shape), one round-robin step's pairs")
        self.m, self.n = 32768, 8192
        gen = torch.Generator(device="cuda")
        gen.manual_seed(5 + rank)
        self.G = torch.randn((self.n, self.m), dtype=torch.float64, device="cuda",
                             generator=gen).T
        self.pairs = J.strategy_pairs(self.n, self.n, 0).contiguous()
        self.ce, self.cf = J.colnorms(self.G)
        self.a21 = torch.rand(self.n // 2, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
        self.units_per_step = self.n // 2
        self.kernel = "dgsscl_kernel"
        self.l2_note = "G 2.1 GB >> L2"

    def prepare(self):
        pass

    def step(self, stream):
        import paper_2202_08361_b200 as J
        J.dgsscl(self.G, self.pairs, self.ce, self.cf, self.a21, stream=stream)

    def bytes_per_step(self):
        return (self.n // 2) * 3 * self.m * 8

    def e2e(self, stream, steps):
        import torch
        import paper_2202_08361_b200 as J
        hG = torch.empty((self.n, self.m), dtype=torch.float64).pin_memory()
        hG.copy_(self.G.T)
        Gt = torch.empty((self.n, self.m), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            Gt.copy_(hG, non_blocking=True)
            J.dgsscl(Gt.T, self.pairs, self.ce, self.cf, self.a21, stream=stream)
            hG.copy_(Gt, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), hG.numel() * 8, hG.numel() * 8

    def cpu_sample(self):
        import oracle as O
        k = 64
        G = self.G[:, :2 * k].cpu().numpy()
        ce, cf = self.ce.cpu().numpy(), self.cf.cpu().numpy()
        a = self.a21.cpu().numpy()

        def run():
            for l in range(k):
                O.dgsscl(G[:, 2 * l], G[:, 2 * l + 1], ce[2 * l], cf[2 * l], ce[2 * l + 1],
                         cf[2 * l + 1], a[l])
        return run, k, f"{k} pairs of 32768 rows per call"


WORKLOADS = {"evd_c64": EvdWorkload, "evd_r64": EvdWorkload, "evd_c32": EvdWorkload, "step_r64": StepWorkload,
             "gesvj_r64": GesvjWorkload, "batched_c64": BatchedWorkload,
             "step_c64": StepC64Workload, "dist_c64": DistC64Workload, "norm_c64": NormWorkload,
             "gs_r64": GsWorkload}


def cpu_baseline(wl, target_s=10.0):
    """The oracle (never tuned) on this box's host cores: the bounded sample
    repeated for ~target_s seconds of CPU work (the contract's 10-30 s)."""
    import oracle as O
    fn, units, what = wl.cpu_sample()
    t0 = time.perf_counter()
    reps = 0
    while True:
        fn()
        reps += 1
        if time.perf_counter() - t0 > target_s or reps >= 100000:
            break
    dt = time.perf_counter() - t0
    out = {"value": units * reps / dt, "unit": wl.unit, "cores": O.num_threads(),
           "kind": "oracle", "sample": f"{what} x {reps} calls ({dt:.1f} s)"}
    if isinstance(wl, EvdWorkload):  # also one core for configs 1-2
        nt = O.num_threads()
        O.set_num_threads(1)
        t0, reps1 = time.perf_counter(), 0
        while time.perf_counter() - t0 < target_s / 4 and reps1 < 100000:
            fn()
            reps1 += 1
        dt1 = time.perf_counter() - t0
        O.set_num_threads(nt)
        out["value_1core"] = units * reps1 / dt1
    return out


def run_jsvd(args):
    import torch
    import paper_2202_08361_b200 as J

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = WORKLOADS[args.workload](args.workload, rank, world)
    stream = torch.cuda.current_stream()
    per_step_events = args.workload in ("batched_c64", "gesvj_r64", "dist_c64")

    for _ in range(args.warmup):
        wl.prepare()
        wl.step(stream)
    torch.cuda.synchronize()
    if hasattr(wl, "reset_counters"):
        wl.reset_counters()
    # steps that are pure asynchronous launches (no host sync, no per-step
    # preparation) are captured once as a CUDA graph of exactly K steps and
    # timed as one replay: the device time of the K launches without the
    # Python/ctypes enqueue cost between them
    graph = None
    if getattr(wl, "graphable", False) and not args.no_graph:  # per rank, no collective inside
        graph = torch.cuda.CUDAGraph()
        nc0 = J.launch_count()
        with torch.cuda.graph(graph):
            cap = torch.cuda.current_stream()
            for _ in range(args.steps):
                wl.step(cap)
        graph_launches = J.launch_count() - nc0
        torch.cuda.synchronize()
        # the first launch of an instantiated graph carries one-time costs (its
        # upload to the device), which are not the steps': upload it untimed
        warm = os.environ.get("JSVD_BENCH_GRAPH_WARM", "upload")
        if warm == "upload":
            graph_upload(graph, stream)
        elif warm == "replay":
            graph.replay()
        torch.cuda.synchronize()
        if hasattr(wl, "reset_counters"):
            wl.reset_counters()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = J.launch_count()
    evs = []
    with ClockSampler(local) as clk:
        if graph is not None:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            graph.replay()
            b.record(stream)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
        elif per_step_events:  # preparation (L2 flush / input restore) outside the timing
            for _ in range(args.steps):
                wl.prepare()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                wl.step(stream)
                b.record(stream)
                evs.append((a, b))
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs)
        else:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                wl.step(stream)
            b.record(stream)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
    launches = J.launch_count() - n0
    if graph is not None:
        launches = graph_launches  # the replay launches exactly the captured kernels
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_per_step = ms / args.steps
    value = world * wl.units_per_step * args.steps / (ms / 1e3)
    if isinstance(wl, GesvjWorkload):
        extra_g = {"sweeps": wl.last["sweeps"], "status": wl.last["status"],
                   "transforms_per_sweep": wl.last["tps"]}

    peak, peak_src = load_peaks()
    extra = {}
    if isinstance(wl, StepWorkload):  # (StepC64Workload included)
        transformed = int(wl.t.item())
        bytes_step = wl.bytes_for(args.steps, transformed) / args.steps
        extra["transformed_pairs_per_step"] = transformed / args.steps
    elif isinstance(wl, DistC64Workload):  # per-GPU share; first sweep: every pair transforms
        bytes_step = wl.bytes_per_step()
        extra.update(sweep_steps_per_call=wl.max_steps, exchange_after_step=wl.max_steps - 2,
                     transforms_first_sweep=wl.last["tps"], status=wl.last["status"])
    else:
        bytes_step = wl.bytes_per_step()
    achieved = bytes_step / (ms_per_step / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": load_traffic(args.workload),
                "peak_source": peak_src, "kernel": wl.kernel,
                # SURVEY 8(d).1 reports both: the measured copy peak and the nominal ~8 TB/s
                "nominal_peak": 8000.0, "nominal_frac": achieved / 8000.0}
    if args.workload in ("step_r64", "gesvj_r64"):
        # configs[2]'s G + V (40 MB) stay in the 126 MB L2 across steps, so the
        # HBM fraction is not the bound: the same algorithmic bytes against a
        # measured L2-resident copy rate (same footprint), as the ceiling
        # ceiling -- the line's roofline; the HBM figures stay beside it
        l2 = l2_resident_copy(40 << 20)
        roofline = {"bound": "l2", "achieved": achieved, "peak": l2, "unit": "GB/s",
                    "frac": achieved / l2, "traffic": roofline["traffic"],
                    "peak_source": "measured: torch copy_ of a 20 MB buffer into another (40 MB, "
                                   "L2-resident), read + write bytes, CUDA graph of 200 copies",
                    "kernel": wl.kernel, "hbm_peak": peak, "hbm_frac": achieved / peak,
                    "hbm_peak_source": peak_src}
    if isinstance(wl, EvdWorkload) and wl.nsets > 1:  # the short configs[0] launch
        extra["size_matched_copy"] = size_matched_copy(wl, args.steps, peak)
    if isinstance(wl, EvdWorkload) and wl.nsets == 1 and not wl.f32:
        extra["streaming_copy"] = streaming_copy(wl, args.steps, peak, achieved)
    if isinstance(wl, GesvjWorkload):
        extra.update(extra_g)
        # capped (ENOCONV): sigma holds Sigma' in column order,
        # Sigma = 2^-scale Sigma' sorted; converged: sigma sorted already
        s = wl.last["sigma"].cpu().numpy()
        if wl.last["status"] != 0:
            s = np.sort(np.ldexp(s, -wl.last["scale"]))[::-1]
        extra["sigma_err_normwise"] = float(np.abs(s - wl.sig_true).max() / wl.sig_true[0])
    if isinstance(wl, BatchedWorkload):
        sw = wl.sw.float().mean().item()
        extra["mean_sweeps"] = sw
        extra["all_converged"] = bool((wl.st == 0).all().item())
        extra["hbm_roofline_frac"] = achieved / peak
        extra["transformed_pair_steps_per_matrix"] = float(wl.tr.double().mean().item())
        # the paper's Fig 5.4 breakdown for this kernel (jsvd_batched_phase_profile,
        # a clock64-instrumented build of the same kernel, run after the timing)
        wl.prepare()
        pr = J.batched_phase_profile(wl.A.transpose(1, 2), stream=stream)
        torch.cuda.synchronize()
        extra["phase_breakdown"] = {
            who: {k: round(v / max(d["sweep loop"], 1), 4) for k, v in d.items() if k != "sweep loop"}
            for who, d in pr.items()}
        # FP64-pipe-bound kernel: algorithmic FP64 operations per second vs the
        # measured DFMA throughput of jsvd_fp64_peak
        ops = wl.fp64_ops()
        ach = ops / (ms_per_step / 1e3)
        fpk = J.fp64_peak(stream=stream)
        roofline = {"bound": "fp64", "achieved": ach / 1e12, "peak": fpk / 1e12,
                    "unit": "T FP64-op/s", "frac": ach / fpk, "traffic": None,
                    "peak_source": "measured: jsvd_fp64_peak (DFMA chains on every SM, this run)",
                    "derived_peak": FP64_PEAK_INSTR / 1e12, "kernel": wl.kernel,
                    "ops_per_step": ops}

    # SURVEY 8(d).4 asks for the median and the best too: per-step times of the
    # timed steps where they exist, else 5 more replays of the K-step graph
    # (after the timed region and after the counters above were read)
    step_stats = None
    if evs:
        per = sorted(a.elapsed_time(b) for a, b in evs)
        step_stats = {"median_ms": per[len(per) // 2], "best_ms": per[0],
                      "source": "per-step CUDA events of the timed steps"}
    elif graph is not None:
        per = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            graph.replay()
            b.record(stream)
            torch.cuda.synchronize()
            per.append(a.elapsed_time(b) / args.steps)
        per.sort()
        step_stats = {"median_ms": per[2], "best_ms": per[0],
                      "source": "5 more replays of the K-step graph, per-step mean of each"}
    e2e_steps = max(1, min(args.steps, 3))
    ems, h2d, d2h = wl.e2e(stream, e2e_steps)
    if dist:
        t = torch.tensor([ems], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    e2e_val = world * wl.units_per_step * e2e_steps / (ems / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl)

    if rank == 0:
        line = {
            "metric": BASELINE_METRIC,
            "value": value,
            "unit": wl.unit,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32" if getattr(wl, "f32", False) else "f64",
            "data": "synthetic (counter-based SplitMix64, DESIGN.md recipe)",
            "config": {"workload": wl.desc, "units_per_gpu_step": wl.units_per_step,
                       "timing": ("one CUDA-graph replay of the K steps (CUDA events)" if graph is not None
                                  else "per-step CUDA events" if per_step_events else
                                  "CUDA events around K launches"),
                       "parallelism": (("column-block shard x%d (B=16, NCCL send/recv in libjsvd)" % world)
                                       if isinstance(wl, DistC64Workload) else
                                       ("batch-index shard x%d of the configured batch" % world))
                       if world > 1 else "single GPU",
                       "l2": wl.l2_note},
            "e2e": {"value": e2e_val, "unit": wl.unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "path": getattr(wl, "e2e_note",
                                    "pinned host copies around the C-ABI device entry, one stream")},
            "gpu_launches": launches,
            "step_stats": step_stats,
            "roofline": roofline,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        line.update(extra)
        emit(line)
    if dist:
        dist.destroy_process_group()


def graph_upload(graph, stream):
    """cuGraphUpload of a captured torch CUDA graph (driver API, no launch)."""
    import ctypes as ct
    cu = ct.CDLL("libcuda.so.1")
    cu.cuGraphUpload.restype = ct.c_int
    cu.cuGraphUpload.argtypes = [ct.c_void_p, ct.c_void_p]
    rc = cu.cuGraphUpload(ct.c_void_p(graph.raw_cuda_graph_exec()), ct.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"cuGraphUpload failed ({rc})")


def l2_resident_copy(footprint):
    """GB/s (read + write bytes) of a device copy whose source and destination
    (footprint bytes together) fit in L2, replayed 200 times in a CUDA graph."""
    import torch
    half = footprint // 2 // 8
    a = torch.ones(half, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    b.copy_(a)
    reps = 200
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            b.copy_(a)
    torch.cuda.synchronize()
    graph_upload(g, torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return reps * 2 * half * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9


def size_matched_copy(wl, steps, peak):
    """Context for the EVD's roofline fraction: a plain device copy (torch
    copy_, read B/2 + write B/2 bytes per step, B = the EVD's algorithmic bytes)
    cycling the same number of buffer sets, K steps in one CUDA graph -- what a
    trivially memory-bound launch of this size reaches on this GPU."""
    import torch
    half = int(wl.bytes_per_step() // 2) // 8
    sets = [(torch.empty(half, dtype=torch.float64, device="cuda").fill_(1.0),
             torch.empty(half, dtype=torch.float64, device="cuda")) for _ in range(wl.nsets)]
    for s_, d_ in sets:
        d_.copy_(s_)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for k in range(steps):
            d_, s_ = sets[k % len(sets)][1], sets[k % len(sets)][0]
            for o in range(0, half, 1 << 27):  # <= 1 GiB slices: 32-bit-indexed copy kernels
                d_[o:o + (1 << 27)].copy_(s_[o:o + (1 << 27)])
    torch.cuda.synchronize()
    graph_upload(g, torch.cuda.current_stream())  # untimed: the first launch carries the upload
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    ach = 2 * half * 8 / (ms / 1e3) / 1e9
    del sets, g
    torch.cuda.empty_cache()
    return {"achieved": ach, "frac": ach / peak, "ms_per_step": ms,
            "what": "torch copy_ of the same bytes (read B/2 + write B/2), same buffer-set cycling"}


def streaming_copy(wl, steps, peak, achieved):
    """Context for the configs[1] line: the library's plain streaming copy
    (jsvd_copy16: the EVD kernel's 16-byte streaming access pattern and
    programmatic dependent launch) of the same bytes per step (read B/2 +
    write B/2), K launches back to back in one CUDA graph as the EVD line
    itself -- the rate a copy sustains over the same window."""
    import torch
    import paper_2202_08361_b200 as J
    n16 = int(wl.bytes_per_step() // 2) // 16
    src = torch.ones(2 * n16, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    J.copy16(src, dst)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cap = torch.cuda.current_stream()
        for _ in range(steps):
            J.copy16(src, dst, stream=cap)
    torch.cuda.synchronize()
    graph_upload(g, torch.cuda.current_stream())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    ach = 2 * n16 * 16 / (ms / 1e3) / 1e9
    del src, dst, g
    torch.cuda.empty_cache()
    return {"achieved": ach, "frac": ach / peak, "ms_per_step": ms, "evd_over_copy": achieved / ach,
            "what": "jsvd_copy16 of the same bytes (read B/2 + write B/2), K launches in one graph"}


def run_reference(args):
    """--impl reference: the oracle on host cores (rank 0 only under torchrun)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle as O
    wl = ReferenceWorkload(args.workload)
    for _ in range(args.warmup):
        wl.fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.fn()
    dt = time.perf_counter() - t0
    v = wl.units * args.steps / dt
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": v, "unit": wl.unit,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if args.workload == "evd_c32" else "f64",
        "data": "synthetic",
        "config": {"workload": wl.desc, "sample_per_step": wl.what},
        "cpu_baseline": {"value": v, "unit": wl.unit, "cores": O.num_threads(),
                         "kind": "oracle", "sample": wl.what},
        "e2e": {"value": v, "unit": wl.unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


class ReferenceWorkload:
    """Bounded per-step samples of each workload for the oracle arm (no GPU)."""

    def __init__(self, name):
        import oracle as O
        import synth
        if name in ("evd_c64", "evd_r64", "evd_c32"):  # noqa: SIM114
            n = 1 << 18
            if name == "evd_c32":
                a = synth.evd_cfg2_f32(n)
                self.fn = lambda: O.evd2_batched_f32(*a)
            else:
                a = synth.evd_cfg2(n) if name == "evd_c64" else synth.evd_cfg1(n)
                self.fn = lambda: O.evd2_batched(*a)
            self.units, self.unit = n, "EVD/s"
            self.desc = DESC[name]
            self.what = f"{n} matrices of the batch per step"
        elif name in ("step_r64", "gesvj_r64"):
            A, _ = synth.svd_cfg3()
            m, n = A.shape
            s0 = (1022 - int(np.floor(np.log2(m)))) - int(np.floor(np.log2(np.abs(A).max()))) - 1
            G = np.asfortranarray(np.ldexp(A, s0))
            V = np.asfortranarray(np.eye(n))
            R = O.RSpec.make(256, 1, [16, 8, 4, 2, 1, 128, 64, 32])
            pairs = O.strategy_pairs(n, n, 0)
            self.fn = lambda: O.step(G, V, pairs, R)
            self.units, self.unit = 1, "sweep-steps/s"
            self.desc = "BASELINE configs[2]: one sweep step of the 4096x1024 real SVD"
            self.what = "one full step (512 pairs) per step"
        elif name in ("step_c64", "dist_c64"):
            # configs[4]: 16 of the 4096 pairs of a step on CPU-generated columns
            # of the configs[4] length, in the step kernel's reduction order R
            # for m = 32768 complex (W = 2048: 8-CTA clusters of 256 threads)
            rng = np.random.default_rng(5)
            m, npairs = 32768, 16
            G = np.asfortranarray((rng.standard_normal((m, 2 * npairs)) +
                                   1j * rng.standard_normal((m, 2 * npairs))) * 2.0 ** 1000)
            V = np.asfortranarray(np.eye(2 * npairs, dtype=np.complex128))
            pairs = np.arange(2 * npairs, dtype=np.int32).reshape(-1, 2)
            R = O.RSpec.make(2048, 1, [16, 8, 4, 2, 1, 128, 64, 32, 1024, 512, 256])
            self.fn = lambda: O.step(G, V, pairs, R)
            self.units, self.unit = npairs / 4096, "sweep-steps/s"
            self.desc = ("BASELINE configs[4]: complex fp64 Jacobi SVD of one 32768x8192 matrix, "
                         "one sweep step")
            self.what = "16 of the 4096 pairs of a step per step (units = fraction of a step)"
        elif name == "gs_r64":
            rng = np.random.default_rng(6)
            m, k = 32768, 64
            G = rng.standard_normal((m, 2 * k))
            ef = [O.norm_ef(G[:, j], s=32) for j in range(2 * k)]
            a = rng.uniform(-1, 1, k)

            def run():
                for l in range(k):
                    O.dgsscl(G[:, 2 * l], G[:, 2 * l + 1], ef[2 * l][0], ef[2 * l][1],
                             ef[2 * l + 1][0], ef[2 * l + 1][1], a[l])
            self.fn = run
            self.units, self.unit = k, "pairs/s"
            self.desc = "NEXT-4 (Alg SM8.1): Gram-Schmidt of g_q against g_p, pairs of 32768 rows"
            self.what = f"{k} pairs of 32768 rows per step"
        elif name == "norm_c64":
            rng = np.random.default_rng(5)
            cols = rng.standard_normal((32768, 4)) + 1j * rng.standard_normal((32768, 4))
            self.fn = lambda: O.norm_ef_cols(cols)
            self.units, self.unit = 4, "columns/s"
            self.desc = DESC["norm_c64"]
            self.what = "4 complex columns of 32768 rows per step"
        else:
            A = synth.svd_cfg4(16)
            R = O.RSpec.make(8, 1, [4, 2, 1])  # the batched kernel's R (m <= 64)
            self.fn = lambda: O.gesvj_batched(A, R)
            self.units, self.unit = 16, "SVD/s"
            self.desc = DESC["batched_c64"]
            self.what = "16 matrices of the batch per step"


def _claim_stdout():
    """stdout carries exactly the JSON line: everything else written to fd 1
    by libraries (NCCL's version banner at communicator creation, ...) goes
    to stderr; returns the stream the JSON line is printed on."""
    sys.stdout.flush()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    return out


JSON_OUT = None


def emit(line):
    print(json.dumps(line), file=JSON_OUT or sys.stdout, flush=True)


def main():
    global JSON_OUT
    JSON_OUT = _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="jsvd", choices=["jsvd", "reference"])
    ap.add_argument("--workload", default="evd_c64", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the K steps as individual launches instead of one CUDA-graph replay")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps is None:
        # (>= ~20 ms timed windows: the clock sampler sees >= 10 samples)
        args.steps = {"evd_c64": 200, "evd_r64": 1600, "evd_c32": 200, "step_r64": 1600, "gesvj_r64": 2,
                      "batched_c64": 3, "step_c64": 50, "dist_c64": 3, "norm_c64": 50,
                      "gs_r64": 50}[args.workload]
    if args.impl == "reference":
        run_reference(args)
    else:
        run_jsvd(args)


if __name__ == "__main__":
    main()
