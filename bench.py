#!/usr/bin/env python3
"""Benchmark driver (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload edge|...]
                    [--impl ours|reference]

Default workload = BASELINE.json configs[1]: edge detection on a batch of 256
synthetic 1080x1920 f32 frames, sharded by frame across ranks (strong
scaling: the 256-frame batch is split).  A "step" is one pass of the hot path
over the batch.

  value  frames/s with inputs resident in HBM (CUDA events on the launching
         stream, barrier + synchronize on both sides, max over ranks)
  e2e    the same metric through the public API with pinned HOST buffers:
         the H2D copy of the frames and the D2H copy of the edge maps are
         inside the timed region
  roofline  dominant kernel (edge_fused): algorithmic bytes per launch
         (8*H*W per frame) / average launch duration, from
         CUDA events recorded by libjunob200 around each launch
  cpu_baseline  the oracle restatement (oracle/, C + OpenMP) on a bounded
         sample, rank 0 at N=1 only

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port, all host threads) on the same metric; only rank 0 works.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


def load_traffic(workload):
    """dram read+write bytes per launch of the workload's dominant kernel, from
    the committed `ncu --set full` capture (profiles/ncu_traffic.json, written by
    tools/ncu_summary.py --json); None when absent"""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f)[workload]
        return e["dram_bytes_per_launch"], e["source"]
    except Exception:
        return None, None


def load_issue(workload):
    """the same capture's issue picture (what binds a kernel that is not at
    its memory or tensor roof): issue-active %, FMA-pipe %, tensor-pipe %"""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f)[workload]
        out = {k: e[k] for k in ("issue_active_pct", "fma_pipe_pct", "tensor_pipe_pct", "warp_inst") if k in e}
        return out or None
    except Exception:
        return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured"
        return d
    except Exception:
        return dict(PEAKS_FALLBACK)


# ------------------------------------------------------------------ dist env
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Dist:
    def __init__(self, backend="nccl"):
        self.rank, self.world, self.local = dist_env()
        self.backend = backend
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist
            # every rank of the launch is in the group the collectives use
            assert dist.get_world_size() == self.world, (dist.get_world_size(), self.world)

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        on_gpu = torch.cuda.is_available() and self.backend == "nccl"
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    def __init__(self, index=0, period=0.005):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _names(self, mask):
        nv = self.nv
        table = {
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        return {k for k, v in table.items() if mask & v}

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                self.reasons |= self._names(fn(self.h))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "note": "nvml unavailable"}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ workloads
class EdgeWorkload:
    name = "edge"
    metric = "edge_detection_frames_per_s"
    unit = "frames/s"
    kernel = "edge_fused"

    def __init__(self, args, rank, world):
        from paper_2503_10855_b200 import workloads as W
        self.batch, self.n, self.m = args.batch, 1080, 1920
        if args.small:
            self.batch, self.n, self.m = 8, 270, 480
        per = [self.batch // world + (1 if r < self.batch % world else 0) for r in range(world)]
        self.local = per[rank]
        self.first = sum(per[:rank])
        self.filters = W.edge_filters()
        self.frames_host = W.edge_batch(self.local, self.n, self.m, seed=1000 + self.first) \
            if self.local else np.zeros((0, self.n, self.m), np.float32)
        self.frame_bytes = self.n * self.m * 4
        self.inst_unit = ("px", self.n * self.m)

    def config(self, world):
        return {"workload": f"edge_detection batch={self.batch} frames {self.n}x{self.m} f32, gs=7 sz=3 sb=3",
                "global_batch": self.batch, "frame": [self.n, self.m], "parallelism": f"frames/{world}",
                "l2": "inputs (2.1 GB) exceed the 126 MB L2; no flush needed"}

    def units_per_step(self):
        return self.batch

    def algorithmic_bytes_per_unit(self):
        return 8 * self.n * self.m  # read input + write edge map once

    def setup_device(self, torch):
        from paper_2503_10855_b200 import _lib
        self.lib = _lib.load()
        self.x = torch.from_numpy(self.frames_host).cuda()
        self.out = torch.empty_like(self.x)
        self.f = [torch.from_numpy(a).cuda() for a in self.filters[:4]]
        self.theta = float(self.filters[4])
        self.stream = torch.cuda.current_stream()
        self.pin_in = torch.from_numpy(self.frames_host).pin_memory() if self.local else None
        self.pin_out = torch.empty(self.frames_host.shape, dtype=torch.float32).pin_memory() \
            if self.local else None

    def step_device(self):
        if not self.local:
            return
        g, st, sx, sy = self.f
        rc = self.lib.jb_edge_f32(self.local, self.n, self.m, 7, 3, 3, self.x.data_ptr(), g.data_ptr(),
                                  st.data_ptr(), sx.data_ptr(), sy.data_ptr(), self.theta,
                                  self.out.data_ptr(), self.stream.cuda_stream)
        if rc:
            from paper_2503_10855_b200 import _lib
            raise RuntimeError(_lib.last_error())

    def step_e2e(self):
        """The public entry on numpy host arrays: api.execute copies the batch
        in, runs the kernel and returns a fresh numpy result every step."""
        if not self.local:
            return
        from paper_2503_10855_b200 import api
        self.e2e_out = api.execute("edge_detection", [self.n, self.m, 7, 3, 3],
                                   [self.frames_host, *self.filters[:4], self.theta])

    def e2e_bytes(self):
        # D2H: the edge maps cross PCIe bit-packed (ceil(n*m/32) words per
        # frame) and are expanded to f32 on the host inside the timed call
        return self.local * self.frame_bytes, self.local * ((self.n * self.m + 31) // 32) * 4

    e2e_api = ("paper_2503_10855_b200.api.execute('edge_detection', ...) on numpy in/out "
               "(input page-locked in place on first use, chunks of 16 frames overlap H2D/kernel/D2H; "
               "maps cross PCIe bit-packed and are expanded to the f32 result on the host thread pool)")

    def ref_step(self, oracle, sample=False):
        """The step on the host: the oracle restatement over the whole batch
        (threads split the frames), or a 32-frame sample of it."""
        k = min(32, self.batch) if sample else self.batch
        g, st, sx, sy, th = self.filters
        x = self.frames_host[:k] if self.local >= k else \
            __import__("paper_2503_10855_b200.workloads", fromlist=["x"]).edge_batch(k, self.n, self.m)
        oracle.edge(x, g, st, sx, sy, th)
        return k, f"{k} frames {self.n}x{self.m} through oracle/juno_oracle.c (OpenMP over frames)"

    def check(self, oracle):
        """Bit-exact spot check of one output frame against the oracle."""
        if not self.local:
            return True
        g, st, sx, sy, th = self.filters
        ref = oracle.edge(self.frames_host[:1], g, st, sx, sy, th)[0]
        got = self.out[0].cpu().numpy()
        ok = bool(np.array_equal(ref.view(np.uint32), got.view(np.uint32)))
        e2e = getattr(self, "e2e_out", None)
        if e2e is not None:  # the end-to-end result (bit-packed D2H + host expansion) too
            ok = ok and bool(np.array_equal(ref.view(np.uint32), np.asarray(e2e[0]).view(np.uint32)))
            ok = ok and bool(np.array_equal(np.asarray(e2e[-1]).view(np.uint32),
                                            self.out[-1].cpu().numpy().view(np.uint32)))
        return ok


class MatmulWorkload:
    """matmul<1024,1024,1024> (BASELINE configs[0]); one step = one
    jb_matmul_f32 call (tf32 split + tcgen05 GEMM).  L2 is flushed before
    every timed call (inputs are 8 MB, far below the 126 MB L2)."""
    name = "matmul"
    metric = "matmul_f32_1024_ms"
    unit = "ms"
    higher_is_better = False
    kernel = "matmul_tcgen05"
    bound = "tensor"
    flush_l2 = True

    def __init__(self, args, rank, world):
        from paper_2503_10855_b200 import dist as D
        from paper_2503_10855_b200 import workloads as W
        self.n = self.m = self.l = 1024
        self.a, self.b = W.matmul_inputs(self.n, self.m, self.l)
        self.local = 1
        # N > 1: row blocks of A and C (dist.MatmulRowBlocks), B broadcast once
        self.world = world
        self.r0, self.rows = D.row_block(self.n, world, rank)
        if world > 1:
            self.scaling = "strong"

    def config(self, world):
        return {"workload": "matmul<1024,1024,1024> f32 (Fig. 1 entry), 3xTF32 tcgen05",
                "parallelism": "single GPU" if world == 1 else
                f"row blocks/{world}: A and C rows split, B broadcast once at setup (dist.MatmulRowBlocks)",
                "l2": "flushed (256 MiB write) before every timed call"}

    def units_per_step(self):
        return 1

    def flops_per_unit(self):
        return 2.0 * self.n * self.m * self.l

    def setup_device(self, torch):
        from paper_2503_10855_b200 import _lib
        from paper_2503_10855_b200 import dist as D
        self.lib = _lib.load()
        self.da = torch.from_numpy(np.ascontiguousarray(self.a[self.r0:self.r0 + self.rows])).cuda()
        self.db = torch.from_numpy(self.b).cuda()
        if self.world > 1:
            self.blocks = D.MatmulRowBlocks(self.db, self.n)   # the one broadcast of B
        self.dc = torch.empty((self.rows, self.l), dtype=torch.float32, device="cuda")
        self.stream = torch.cuda.current_stream()
        self.pa = torch.from_numpy(self.a).pin_memory()
        self.pb = torch.from_numpy(self.b).pin_memory()
        self.pc = torch.empty((self.n, self.l), dtype=torch.float32).pin_memory()

    def step_device(self):
        rc = self.lib.jb_matmul_f32(self.rows, self.m, self.l, self.da.data_ptr(), self.db.data_ptr(),
                                    self.dc.data_ptr(), self.stream.cuda_stream)
        if rc:
            from paper_2503_10855_b200 import _lib
            raise RuntimeError(_lib.last_error())

    def step_e2e(self):
        from paper_2503_10855_b200 import api
        a = self.a if self.world == 1 else self.a[self.r0:self.r0 + self.rows]
        self.e2e_out = api.execute("matmul", [a.shape[0], self.m, self.l], [a, self.b])

    e2e_api = "paper_2503_10855_b200.api.execute('matmul', ...) on numpy in/out"

    def e2e_bytes(self):
        return 4 * (self.rows * self.m + self.m * self.l), 4 * self.rows * self.l

    def ref_step(self, oracle, sample=False):
        oracle.matmul(self.a, self.b)
        return 1, "the full 1024x1024x1024 call, oracle/juno_oracle.c (OpenMP over rows)"

    def check(self, oracle):
        ref = oracle.matmul(self.a, self.b)
        got = self.dc.cpu().numpy()
        return bool(np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-5)


class _DeviceCall:
    """Shared plumbing for the single-call workloads below: host arrays are
    uploaded once (value), or copied H2D + D2H around every call (e2e)."""
    flush_l2 = False
    scaling = "weak"
    local = 1

    def setup_device(self, torch):
        from paper_2503_10855_b200 import _lib
        self.torch = torch
        self.lib = _lib.load()
        self.stream = torch.cuda.current_stream()
        self.dev = {}
        self.pin = {}
        for k, a in self.host.items():
            t = torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a)
            self.dev[k] = t.cuda()
            self.pin[k] = t.pin_memory()
        self.alloc_outputs(torch)

    def check_rc(self, rc):
        if rc:
            from paper_2503_10855_b200 import _lib
            raise RuntimeError(_lib.last_error())

    def step_e2e(self):
        if getattr(self, "world", 1) == 1 and hasattr(self, "execute_args"):
            # the public entry on numpy host arrays (fresh numpy results)
            from paper_2503_10855_b200 import api
            entry, dcs, args = self.execute_args()
            self.e2e_out = api.execute(entry, dcs, args)
            return
        for k in self.inputs_e2e:
            self.dev[k].copy_(self.pin[k], non_blocking=True)
        self.step_device()
        for k, t in self.outputs_e2e():
            self.pin_out[k].copy_(t, non_blocking=True)
        self.stream.synchronize()

    @property
    def e2e_api(self):
        if getattr(self, "world", 1) == 1 and hasattr(self, "execute_args"):
            return f"paper_2503_10855_b200.api.execute('{self.execute_args()[0]}', ...) on numpy in/out"
        return "pinned host buffers around the sharded step"

    def e2e_bytes(self):
        h2d = sum(self.host[k].nbytes for k in self.inputs_e2e)
        d2h = sum(t.numel() * t.element_size() for _, t in self.outputs_e2e())
        return h2d, d2h


class SradWorkload(_DeviceCall):
    """srad<16384,16384>(niter=10, lambda=0.5): one step = one call."""
    name = "srad"
    metric = "srad_16384x16384_ms_per_iteration"
    unit = "ms"
    higher_is_better = False
    kernel = "srad_iter"
    bound = "hbm"
    niter = 100

    def __init__(self, args, rank, world):
        from paper_2503_10855_b200 import dist as D
        from paper_2503_10855_b200 import workloads as W
        self.rows = self.cols = 4096 if args.small else 16384
        img = W.srad_image(self.rows, self.cols)
        # N > 1: row slabs of one image (strong scaling), NCCL halo exchange
        # of the J rows + allreduce of the f64 statistics per iteration
        self.world = world
        self.plan = D.srad_slab(self.rows, world, rank)
        self.own_rows = self.plan["r1"] - self.plan["r0"]
        if world > 1:
            img = np.ascontiguousarray(img[self.plan["r0"]:self.plan["r1"]])
            self.scaling = "strong"
        self.host = {"image": img}
        self.inputs_e2e = ["image"]

    def alloc_outputs(self, torch):
        self.out = torch.empty((self.own_rows, self.cols), dtype=torch.float32, device="cuda")
        self.pin_out = {"out": torch.empty((self.own_rows, self.cols), dtype=torch.float32).pin_memory()}
        if self.world > 1:
            from paper_2503_10855_b200 import dist as D
            self.be = D.CudaSradBackend()
            # default: the fused peer-memory step (one kernel per iteration,
            # boundary rows and sums stored into the peers over NVLink);
            # JB_SRAD_NCCL=1 selects the NCCL halo + allreduce path
            self.slabs = None
            if os.environ.get("JB_SRAD_NCCL") != "1":
                self.slabs = D.SradP2PSlabs(self.rows, self.cols, grid=int(os.environ.get("JB_SRAD_P2P_GRID", "0")))

    def outputs_e2e(self):
        return [("out", self.out)]

    def config(self, world):
        fused = getattr(self, "slabs", None) is not None
        par = "single GPU" if world == 1 else (
            f"row slabs/{world}: " + ("fused P2P step (peer-memory halo rows + mailbox sums)" if fused
                                      else "NCCL halo rows + f64 allreduce per iteration"))
        return {"workload": f"srad<{self.rows},{self.cols}> niter={self.niter} lambda=0.5 (Rodinia srad_v1)",
                "parallelism": par, "l2": "1 GiB image >> 126 MB L2"}

    def units_per_step(self):
        return self.niter

    def algorithmic_bytes_per_unit(self):
        # read J + write J' per iteration, of this rank's rows
        return 8 * self.own_rows * self.cols

    def step_device(self):
        if self.world > 1:
            from paper_2503_10855_b200 import dist as D
            if self.slabs is not None:
                res = D.srad_distributed_p2p(self.dev["image"], self.niter, 0.5, self.slabs, self.be)
            else:
                res = D.srad_distributed(self.dev["image"], self.niter, 0.5, self.rows, self.cols, self.be)
            self.out.copy_(res)
            return
        self.check_rc(self.lib.jb_srad_f32(self.rows, self.cols, self.niter, 0.5, self.dev["image"].data_ptr(),
                                           self.out.data_ptr(), None, self.stream.cuda_stream))

    def value_from(self, ms_per_step):
        return ms_per_step / self.niter

    def execute_args(self):
        return "srad", [self.rows, self.cols], [self.niter, 0.5, self.host["image"]]

    def ref_step(self, oracle, sample=False):
        oracle.srad(self.host["image"], 1, 0.5)
        return 1, f"1 iteration (with extract + compress) of the full {self.rows}x{self.cols} image"

    def check(self, oracle):
        crop = np.ascontiguousarray(self.host["image"][:512, :512])
        import paper_2503_10855_b200 as jbp
        got = jbp.srad(3, 0.5, crop)
        ref = oracle.srad(crop, 3, 0.5)
        return bool(np.allclose(got, ref, rtol=1e-4, atol=1e-4))


class EulerWorkload(_DeviceCall):
    """euler<2^22> on a 2048x2048 structured-synthetic mesh, 10 iterations
    (3 RK stages each) per step."""
    name = "euler"
    metric = "cfd_euler_2048x2048_ms_per_iteration"
    unit = "ms"
    higher_is_better = False
    kernel = "euler_rk"
    bound = "hbm"
    iters = 10

    def __init__(self, args, rank, world):
        from paper_2503_10855_b200 import dist as D
        from paper_2503_10855_b200 import workloads as W
        self.w = self.h = 512 if args.small else 2048
        areas, nb, normals, ff, v = W.euler_mesh(self.w, self.h)
        self.nelr = areas.shape[0]
        self.world = world
        self.n_own = self.nelr
        if world > 1:
            # element-range slabs of one mesh (strong scaling): slab-local
            # neighbour ids, NCCL halo exchange of the stage input per RK stage
            self.plans = D.euler_plans(nb, world)
            self.plan = self.plans[rank]
            self.mesh_nb = nb
            e0, e1 = self.plan["e0"], self.plan["e1"]
            self.n_own = e1 - e0
            vl = np.zeros((5, self.plan["n_loc"]), np.float32)
            vl[:, :self.n_own] = v[:, e0:e1]
            areas, normals, v = (np.ascontiguousarray(areas[e0:e1]), np.ascontiguousarray(normals[:, :, e0:e1]), vl)
            nb = self.plan["neighbors"]
            self.scaling = "strong"
        self.host = {"areas": areas, "nb": nb, "normals": normals, "ff": ff, "v": v}
        self.inputs_e2e = ["areas", "nb", "normals", "ff", "v"]

    def alloc_outputs(self, torch):
        self.pin_out = {"v": torch.empty(self.host["v"].shape, dtype=torch.float32).pin_memory()}
        if self.world > 1:
            from paper_2503_10855_b200 import dist as D
            self.be = D.CudaEulerBackend()
            self.plan[("_nbrs", str(self.dev["nb"].device))] = self.dev["nb"]
            # default: the fused peer-memory exchange (stage kernel + push
            # kernel per RK stage); JB_EULER_NCCL=1 selects the NCCL path
            self.slabs = None
            if os.environ.get("JB_EULER_NCCL") != "1":
                self.slabs = D.EulerP2PSlabs(self.mesh_nb, plans=self.plans)
                self.slabs.plan[("_nbrs", str(self.dev["nb"].device))] = self.dev["nb"]

    def outputs_e2e(self):
        return [("v", self.dev["v"])]

    def config(self, world):
        fused = getattr(self, "slabs", None) is not None
        par = "single GPU" if world == 1 else (
            f"element slabs/{world}: " + ("fused P2P (push kernel into peer memory + arrival counters) per RK stage"
                                          if fused else "NCCL halo exchange per RK stage"))
        return {"workload": f"euler<{self.nelr}> {self.w}x{self.h} structured mesh, {self.iters} iterations x RK3",
                "parallelism": par, "l2": f"{self.nelr * 128 / 1e6:.0f} MB streamed per stage > L2"}

    def units_per_step(self):
        return self.iters

    def algorithmic_bytes_per_unit(self):
        # per RK stage and element: own vars 20 + normals 48 + neighbour ids 16
        # + old vars 20 + area 4 + new vars 20 = 128 B (neighbour vars cached)
        return 3 * 128 * self.n_own  # per iteration = 3 RK-stage launches (this rank's elements)

    def step_device(self):
        d = self.dev
        if self.world > 1:
            from paper_2503_10855_b200 import dist as D
            if self.slabs is not None:
                res = D.euler_distributed_p2p(self.slabs, d["areas"], d["normals"], d["ff"],
                                              d["v"][:, :self.n_own], self.iters)
                d["v"][:, :self.n_own].copy_(res)
            else:
                D.euler_distributed(self.plan, d["areas"], d["normals"], d["ff"], d["v"], self.iters, self.be)
            return
        self.check_rc(self.lib.jb_euler_f32(self.nelr, self.iters, d["areas"].data_ptr(), d["nb"].data_ptr(),
                                            d["normals"].data_ptr(), d["ff"].data_ptr(), d["v"].data_ptr(),
                                            self.stream.cuda_stream))

    def value_from(self, ms_per_step):
        return ms_per_step / self.iters

    def execute_args(self):
        h = self.host
        return "euler", [self.nelr], [self.iters, h["areas"], h["nb"], h["normals"], h["ff"], h["v"]]

    def ref_step(self, oracle, sample=False):
        h = self.host
        oracle.euler(h["areas"], h["nb"], h["normals"], h["ff"], h["v"], 1)
        return 1, "1 iteration (3 RK stages) of the full mesh, oracle/juno_oracle.c (OpenMP)"

    def check(self, oracle):
        from paper_2503_10855_b200 import workloads as W
        import paper_2503_10855_b200 as jbp
        m = W.euler_mesh(256, 128, seed=5)
        return bool(np.array_equal(jbp.euler(2, *m, exact=True), oracle.euler(*m, 2)))


class BfsWorkload(_DeviceCall):
    """bfs<2^24, ~6*2^24> from source 0; one step = one traversal."""
    name = "bfs"
    metric = "bfs_16M_gteps"
    unit = "GTEPS"
    higher_is_better = True
    kernel = "bfs_levels"
    bound = "hbm"

    def __init__(self, args, rank, world):
        from paper_2503_10855_b200 import workloads as W
        self.n = 1 << (20 if args.small else 24)
        s, d, e = W.bfs_graph(self.n)
        self.m = e.shape[0]
        self.host = {"s": s, "d": d, "e": e}
        self.inputs_e2e = ["s", "d", "e"]

    def execute_args(self):
        h = self.host
        return "bfs", [self.n, self.m], [h["s"], h["d"], h["e"], 0]

    def alloc_outputs(self, torch):
        self.cost = torch.empty(self.n, dtype=torch.int32, device="cuda")
        self.pin_out = {"cost": torch.empty(self.n, dtype=torch.int32).pin_memory()}

    def outputs_e2e(self):
        return [("cost", self.cost)]

    def config(self, world):
        return {"workload": f"bfs n={self.n} m={self.m} (degree U{{1..11}}, seed 42), source 0",
                "parallelism": "replicas" if world > 1 else "single GPU",
                "l2": "CSR 0.5 GB > L2; visited bitmap (2 MiB) L2-resident by design"}

    def units_per_step(self):
        return self.m / 1e9  # giga-edges

    def algorithmic_bytes_per_unit(self):
        # 8n + 8m bytes per traversal per giga-edge unit
        return (8 * self.n + 8 * self.m) / (self.m / 1e9)

    def step_device(self):
        d = self.dev
        self.check_rc(self.lib.jb_bfs(self.n, self.m, d["s"].data_ptr(), d["d"].data_ptr(), d["e"].data_ptr(), 0,
                                      self.cost.data_ptr(), self.stream.cuda_stream))

    def ref_step(self, oracle, sample=False):
        h = self.host
        oracle.bfs(h["s"], h["d"], h["e"], 0)
        return self.m / 1e9, "the full traversal, oracle/juno_oracle.c (sequential level loop)"

    def check(self, oracle):
        h = self.host
        return bool(np.array_equal(self.cost.cpu().numpy(), oracle.bfs(h["s"], h["d"], h["e"], 0)))


class BackpropWorkload(_DeviceCall):
    """backprop<2^24,16,1>: one bpnn_train step per step."""
    name = "backprop"
    metric = "backprop_16M_train_step_ms"
    unit = "ms"
    higher_is_better = False
    kernel = "bp_adjust"
    bound = "hbm"

    def __init__(self, args, rank, world):
        from paper_2503_10855_b200 import workloads as W
        self.n_in = 1 << (20 if args.small else 24)
        x, iw, hw, t, ipw, hpw = W.bp_inputs(self.n_in, 16, 1)
        self.host = {"x": x, "iw": iw, "hw": hw, "t": t, "ipw": ipw, "hpw": hpw}
        self.inputs_e2e = ["x", "iw", "hw", "t", "ipw", "hpw"]

    def execute_args(self):
        h = self.host
        return "backprop", [self.n_in, 16, 1], [h["x"], h["iw"], h["hw"], h["t"], h["ipw"], h["hpw"]]

    def alloc_outputs(self, torch):
        self.hidden = torch.empty(17, dtype=torch.float32, device="cuda")
        self.output = torch.empty(2, dtype=torch.float32, device="cuda")
        self.errs = torch.empty(2, dtype=torch.float32, device="cuda")
        self.pin_out = {k: torch.empty(self.host[k].shape, dtype=torch.float32).pin_memory()
                        for k in ("iw", "hw", "ipw", "hpw")}
        self.pin_out["errs"] = torch.empty(2, dtype=torch.float32).pin_memory()

    def outputs_e2e(self):
        return [(k, self.dev[k]) for k in ("iw", "hw", "ipw", "hpw")] + [("errs", self.errs)]

    def config(self, world):
        return {"workload": f"backprop<{self.n_in},16,1> one bpnn_train step (Rodinia init)",
                "parallelism": "single GPU", "l2": "weights 2 x 1.07 GiB >> L2"}

    def units_per_step(self):
        return 1

    def algorithmic_bytes_per_unit(self):
        return 16 * (self.n_in + 1) * 17  # adjust_weights: read w, oldw; write w, oldw

    def step_device(self):
        d = self.dev
        self.check_rc(self.lib.jb_bp_train_f32(self.n_in, 16, 1, d["x"].data_ptr(), d["iw"].data_ptr(),
                                               d["hw"].data_ptr(), d["t"].data_ptr(), d["ipw"].data_ptr(),
                                               d["hpw"].data_ptr(), self.hidden.data_ptr(), self.output.data_ptr(),
                                               self.errs.data_ptr(), self.stream.cuda_stream))

    def ref_step(self, oracle, sample=False):
        h = self.host
        oracle.bp_train(h["x"], h["iw"], h["hw"], h["t"], h["ipw"], h["hpw"])
        return 1, f"the full bpnn_train step at n_in={self.n_in}, oracle/juno_oracle.c (OpenMP)"

    def check(self, oracle):
        from paper_2503_10855_b200 import workloads as W
        import paper_2503_10855_b200 as jbp
        x, iw, hw, t, ipw, hpw = W.bp_inputs(4096, 16, 1, seed=9)
        got = jbp.backprop(x, iw, hw, t, ipw, hpw)
        ref = oracle.bp_train(x, iw, hw, t, ipw, hpw)
        return bool(np.allclose(got[2], ref["input_weights"], rtol=1e-6))


class CavaWorkload(_DeviceCall):
    """cava on a batch of 64 synthetic 1080x1920 raw frames, P=16, sharded by
    frame across ranks (strong scaling, no collective)."""
    name = "cava"
    metric = "cava_frames_per_s"
    unit = "frames/s"
    higher_is_better = True
    kernel = "cava_fused"
    bound = "hbm"
    scaling = "strong"

    def __init__(self, args, rank, world):
        from paper_2503_10855_b200 import dist as D
        from paper_2503_10855_b200 import workloads as W
        self.P = args.ctrl_pts
        # P=16: the memory-light variant; thousands of points (the compute
        # variant, e.g. --ctrl-pts 4096) get a smaller batch
        self.batch = 4 if args.small else (64 if self.P <= 64 else 8)
        self.r, self.c = (270, 480) if args.small else (1080, 1920)
        self.inst_unit = ("px", self.r * self.c)
        f0, self.local = D.shard_frames(self.batch, world, rank)
        raw = W.cava_raw(self.batch, self.r, self.c)[f0:f0 + self.local]
        self.host = {"raw": np.ascontiguousarray(raw)}
        self.params = W.cava_params(self.P)
        for k, v in zip(("tstw", "ctrl", "wts", "coefs", "tmap"), self.params):
            self.host[k] = v
        self.inputs_e2e = ["raw"]

    def alloc_outputs(self, torch):
        self.out = torch.empty(self.host["raw"].shape, dtype=torch.uint8, device="cuda")
        self.pin_out = {"out": torch.empty(self.host["raw"].shape, dtype=torch.uint8).pin_memory()}

    def outputs_e2e(self):
        return [("out", self.out)]

    def config(self, world):
        return {"workload": f"cava batch={self.batch} u8[3,{self.r},{self.c}] P={self.P} control points",
                "global_batch": self.batch, "parallelism": f"frames/{world}",
                "l2": f"{self.batch * 6 * self.r * self.c / 1e6:.0f} MB in+out >> 126 MB L2"}

    def units_per_step(self):
        return self.batch

    def algorithmic_bytes_per_unit(self):
        return 6 * self.r * self.c  # u8 x3 in + u8 x3 out

    e2e_api = ("paper_2503_10855_b200.api.execute('cava', ...) on numpy in/out "
               "(input page-locked in place on first use, 8-frame chunks overlap copies and kernels)")

    def step_e2e(self):
        """The public entry on numpy host arrays."""
        from paper_2503_10855_b200 import api
        if self.local:
            self.e2e_out = api.execute("cava", [self.r, self.c, self.P], [self.host["raw"], *self.params])

    def step_device(self):
        if not self.local:
            return
        d = self.dev
        self.check_rc(self.lib.jb_cava_u8(self.local, self.r, self.c, self.P, d["raw"].data_ptr(),
                                          d["tstw"].data_ptr(), d["ctrl"].data_ptr(), d["wts"].data_ptr(),
                                          d["coefs"].data_ptr(), d["tmap"].data_ptr(), self.out.data_ptr(),
                                          self.stream.cuda_stream))

    def ref_step(self, oracle, sample=False):
        k = min(16, self.local) if sample else self.local
        oracle.cava(self.host["raw"][:k], *self.params)
        return k, f"{k} frames, oracle/juno_oracle.c (OpenMP over frames)"

    def check(self, oracle):
        return bool(np.array_equal(self.out[:1].cpu().numpy(), oracle.cava(self.host["raw"][:1], *self.params)))


WORKLOADS = {"edge": EdgeWorkload, "matmul": MatmulWorkload, "srad": SradWorkload, "euler": EulerWorkload,
             "bfs": BfsWorkload, "backprop": BackpropWorkload, "cava": CavaWorkload}


# ------------------------------------------------------------------ arms
def run_ours(args):
    import torch
    rank, world, local = dist_env()
    # JB_BENCH_SHARE_GPU=1 (testing only): every rank on the visible GPU(s)
    # round-robin with a gloo control plane, to exercise the N>1 code path on
    # a one-GPU box; its numbers are not scaling results
    share = os.environ.get("JB_BENCH_SHARE_GPU") == "1"
    torch.cuda.set_device(local % torch.cuda.device_count() if share else local)
    d = Dist("gloo" if share else "nccl")
    from paper_2503_10855_b200 import _lib
    wl = WORKLOADS[args.workload](args, rank, world)
    wl.setup_device(torch)
    dev_stream = torch.cuda.current_stream()
    hib = getattr(wl, "higher_is_better", True)
    flush = getattr(wl, "flush_l2", False)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if flush else None

    def timed(fn, steps):
        """Device ms for `steps` calls; with flush_l2 each call is timed on
        its own event pair after an untimed 256 MiB L2-evicting write."""
        d.barrier()
        torch.cuda.synchronize()
        if not flush:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(dev_stream)
            for _ in range(steps):
                fn()
            e1.record(dev_stream)
            torch.cuda.synchronize()
            d.barrier()
            return e0.elapsed_time(e1)
        evs = []
        for _ in range(steps):
            flush_buf.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(dev_stream)
            fn()
            e1.record(dev_stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        d.barrier()
        return sum(a.elapsed_time(b) for a, b in evs)

    for _ in range(args.warmup):
        wl.step_device()
    torch.cuda.synchronize()

    _lib.prof_reset()
    _lib.prof_enable(True)
    launches0 = _lib.launch_count()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms = timed(wl.step_device, args.steps)
    launches = _lib.launch_count() - launches0
    _lib.prof_enable(False)
    kms, kcount = _lib.prof_read(wl.kernel)
    ms_max = d.max(ms)

    # e2e through the public API (host buffers)
    # e2e warm-up: the first calls page-lock the caller's input arrays and
    # fill the pinned result pool (a caller's steady state holds the previous
    # result while the next call runs: two pool blocks per output)
    for _ in range(max(3, args.warmup // 2)):
        wl.step_e2e()
    torch.cuda.synchronize()
    e2e_ms = d.max(timed(wl.step_e2e, args.e2e_steps))

    units = wl.units_per_step()
    if hib:
        value = units * args.steps / (ms_max / 1e3)
        e2e_value = units * args.e2e_steps / (e2e_ms / 1e3)
    else:  # time-like metric: ms per step (or per unit via value_from)
        vf = getattr(wl, "value_from", lambda x: x)
        value = vf(ms_max / args.steps)
        e2e_value = vf(e2e_ms / args.e2e_steps)
    peaks = load_peaks()
    if args.traffic is None:
        args.traffic, traffic_src = load_traffic(args.workload)
    else:
        traffic_src = "--traffic"
    roofline = None
    if kcount:
        avg_ms = kms / kcount
        # units this rank's kernels processed (frame-sharded workloads: its share)
        local_units = (wl.local if isinstance(wl, (EdgeWorkload, CavaWorkload)) else units) * args.steps
        per_launch_units = local_units / kcount
        if getattr(wl, "bound", "hbm") == "tensor":
            alg = wl.flops_per_unit() * per_launch_units
            ach = alg / (avg_ms / 1e3) / 1e12
            peak = peaks["bf16_tflops"] / 6.0
            roofline = {"kernel": wl.kernel, "bound": "tensor", "achieved": round(ach, 2), "peak": round(peak, 1),
                        "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                        "peak_source": (f"3xTF32 effective = {peaks['source']} bf16 {peaks['bf16_tflops']} "
                                        "TFLOP/s / 2 (tf32 rate) / 3 (three MMAs per product)"),
                        "traffic": args.traffic, "avg_launch_ms": round(avg_ms, 5),
                        "units_per_launch": per_launch_units, "share_of_step": round(kms / ms, 3)}
        else:
            alg = wl.algorithmic_bytes_per_unit() * per_launch_units
            ach = alg / (avg_ms / 1e3) / 1e9
            roofline = {"kernel": wl.kernel, "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"],
                        "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4),
                        "peak_source": f"{peaks['source']} MEASURED_PEAKS.json hbm_gbs",
                        "traffic": args.traffic, "avg_launch_ms": round(avg_ms, 4),
                        "units_per_launch": per_launch_units, "share_of_step": round(kms / ms, 3)}
        roofline["traffic_unit"] = "bytes/launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)"
        roofline["traffic_source"] = traffic_src
        if hasattr(wl, "roofline_extra"):
            roofline.update(wl.roofline_extra(avg_ms, per_launch_units))
        issue = load_issue(args.workload)
        if issue:
            # thread-instructions per unit (instr/px vs FP32
            # issue for the compute-bound stencils); the capture ran this
            # same default configuration, one launch
            wi = issue.pop("warp_inst", None)
            iu = getattr(wl, "inst_unit", None)
            if wi and iu and world == 1 and not args.small:
                issue[f"thread_inst_per_{iu[0]}"] = round(wi * 32 / (per_launch_units * iu[1]), 1)
            if wi and world == 1 and not args.small:
                # the SM issue roofline for the compute-bound kernels: thread
                # instructions per second of this run's launches against one
                # instruction per lane per clock on every SM
                mhz = clk.summary().get("sm_mhz") or 1965.0
                peak_ti = torch.cuda.get_device_properties(0).multi_processor_count * 128 * mhz * 1e6
                ach_ti = wi * 32 / (avg_ms / 1e3)
                issue["issue_roofline"] = {"achieved_tinst_per_s": float(f"{ach_ti:.4g}"),
                                           "peak_tinst_per_s": float(f"{peak_ti:.4g}"),
                                           "frac": round(ach_ti / peak_ti, 3),
                                           "note": "warp instructions from the ncu capture x 32 / live avg launch time"}
            roofline["ncu_issue"] = issue
    h2d, d2h = wl.e2e_bytes()
    res = {"metric": wl.metric, "value": round(value, 4 if not hib else 2), "unit": wl.unit, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
           "higher_is_better": hib, "scaling": getattr(wl, "scaling", "strong"), "vs_baseline": None,
           "dtype": "f32", "data": "synthetic (seeded; paper_2503_10855_b200/workloads.py)",
           "config": wl.config(world),
           "e2e": {"value": round(e2e_value, 4 if not hib else 2), "unit": wl.unit,
                   "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                   "api": getattr(wl, "e2e_api", "public API on pinned host buffers")},
           "roofline": roofline, "gpu_launches": int(launches), "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle
        threads = oracle.max_threads()
        v, _, sample = ref_timed(wl, oracle, warmup=1, steps=3, sample=True)
        res["cpu_baseline"] = {"value": round(v, 4), "unit": wl.unit, "cores": threads, "kind": "port",
                               "sample": sample + "; median of 3 after 1 warm-up"}
        res["parity_spot_check"] = "pass" if wl.check(oracle) else "MISMATCH"
    if rank == 0:
        print(json.dumps(res), flush=True)
    d.close()


def ref_timed(wl, oracle, warmup, steps, sample=False):
    """Time ``steps`` host steps of the workload (after ``warmup``): returns
    (metric value of the median step, median step ms, description)."""
    hib = getattr(wl, "higher_is_better", True)
    times, units, desc = [], 1, ""
    for i in range(warmup + steps):
        t = time.perf_counter()
        units, desc = wl.ref_step(oracle, sample=sample)
        dt = time.perf_counter() - t
        if i >= warmup:
            times.append(dt)
    med = statistics.median(times)
    value = units / med if hib else med * 1e3 / units
    return value, med * 1e3, desc


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle
    wl = WORKLOADS[args.workload](args, 0, 1)
    # every host thread: torch.distributed.run exports OMP_NUM_THREADS=1 to
    # its workers, which would time a single-threaded reference at N > 1
    oracle.set_threads(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
    threads = oracle.max_threads()
    # each step is one real host step (ref_step), timed as it runs: the
    # full batch for edge/CAVA/matmul/BFS/backprop, one iteration of the
    # full grid for SRAD/CFD (their metric is per iteration)
    value, step_ms, desc = ref_timed(wl, oracle, args.warmup, args.steps)
    hib = getattr(wl, "higher_is_better", True)
    res = {"impl": "reference", "metric": wl.metric, "value": round(value, 4), "unit": wl.unit,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 2),
           "higher_is_better": hib,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": dict(wl.config(world), reference_step=desc),
           "cpu_baseline": {"value": round(value, 4), "unit": wl.unit, "cores": threads, "kind": "port",
                            "sample": desc + f"; median of {args.steps} timed steps"},
           "e2e": {"value": round(value, 4), "unit": wl.unit, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "note": "reference CPU path = oracle/juno_oracle.c (C restatement of the Juno program, "
                   "OpenMP); the reference's own interpreter (skiff oracle_execute) "
                   "cannot run these sizes and is pinned to the port by tests/golden"}
    print(json.dumps(res), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--workload", default="edge", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--ctrl-pts", type=int, default=16, help="CAVA control points (16 or e.g. 4096)")
    ap.add_argument("--small", action="store_true", help="tiny config for smoke runs")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch from an ncu capture (profiles/)")
    args = ap.parse_args(argv)
    if args.warmup < 3 and not args.small:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
