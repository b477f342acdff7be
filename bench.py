"""Benchmark of the HAS data plane on B200 (BASELINE.json metric).

Step = one pass of the hot path over one batch of the workload:
  * translate: every owned guest's random-VA batch, one pv_translate launch
    over all owned processes (uncached software translation, the walk
    ProcessTranslator._resolve_page performs; memvirt.py:596-601);
  * copy: every owned guest's copy_to_user op batch through the hybrid
    (hardware HAS) translator: pv_copy_plan + pv_copy_stamp + pv_copy_exec
    (copy_user_buffer semantics, memvirt.py:604-628).
Workload C5 (default, BASELINE configs[4]): 8 shadow guests x 8 GiB, per
guest 16 M random VAs + 1 GiB of 4 MiB copy ops; guest g runs on rank
g mod N (no collective on the data path; "strong" scaling: fixed total work).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
        [--workload c5|c1]
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import ctypes
import hashlib
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

METRIC = "translations/sec and forwarded-copy GB/s (% HBM roofline) at 1/2/4/8 B200 vs CPU ref"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c5", "c1", "c2", "c3", "c4"], default="c5")
    ap.add_argument("--c2-ops", type=int, default=10_000_000)
    ap.add_argument("--c1-mode", choices=["shadow", "tdp", "4l"], default="shadow",
                    help="C1 translator: shadow table (one stage) or guest table + TDP (two stages)")
    ap.add_argument("--scale", type=int, default=1, help="shrink C5 by this factor (testing only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", action="store_true", help="return every guest's translations to rank 0 after "
                    "timing (point-to-point over NCCL = NVLink peer copies) and report its time (default at N > 1)")
    ap.add_argument("--no-gather", action="store_true", help="skip the result return to rank 0 at N > 1")
    ap.add_argument("--no-peer-return", action="store_true", help="C5 at N > 1: the walk writes its lane words "
                    "into local memory instead of straight into rank 0's HBM (shard.PeerResultBuffer); the "
                    "results then return by the separate gather (--gather)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-size parity check against the oracle "
                    "after the timed steps")
    ap.add_argument("--walk-form", choices=["words", "packed", "unpacked"], default="words",
                    help="C5/C1: what the walk writes per lane -- a 4-byte pv_translate_words word + exception "
                    "records (default), a PV_OUT_PACKED u64, or the (u64 value, u32 status) pair; decoded for "
                    "the parity check, and the next form is timed beside it in the same run")
    ap.add_argument("--unpacked", dest="walk_form", action="store_const", const="unpacked",
                    help="same as --walk-form unpacked")
    ap.add_argument("--split-sms", type=int, default=None, help="C5/C1: run the walk on its own partition of at "
                    "least this many SMs beside plan + exec on the rest (green contexts, pv_sm_split); 0 = phases "
                    "back to back (default: 64 for C5 -- the best of 40-72 on one B200, scripts/split_sweep.sh --, "
                    "0 otherwise); value and the rooflines always come from K steps with the phases back to back")
    ap.add_argument("--overlap", action="store_true", help="time C5/C1 steps with the walk on a second stream "
                    "beside plan + exec (A/B option: measured slower than back-to-back phases, "
                    "profiles/r02_overlap_ab.md)")
    ap.add_argument("--no-graph", action="store_true", help="launch the C5 step phases eagerly instead of "
                    "replaying CUDA graphs of them")
    ap.add_argument("--cpu-sample-vas", type=int, default=128 << 20,
                    help="translations the CPU legs time per step (default: all of C5's 128 M)")
    ap.add_argument("--cpu-sample-bytes", type=int, default=8 << 30,
                    help="copy_to_user bytes the CPU legs time per step (default: all of C5's 8 GiB)")
    return ap.parse_args()


def _pg() -> bool:
    """A process group exists (torchrun); PV_BENCH_EMULATE=1 runs one rank's
    share of an N-rank job alone (RANK / WORLD_SIZE set by hand, no group):
    per-rank timing estimates on a one-GPU box, no max over ranks."""
    import torch.distributed as tdist

    return tdist.is_available() and tdist.is_initialized()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PV_BENCH_SHARED_DEVICE") == "1":
        local = 0  # testing only: every rank on cuda:0 (exercises the N>1 path on a one-GPU box, over gloo)
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class L2Flush:
    """Evicts the L2 between timed steps of the workloads whose inputs fit in
    it (C1, C3, C4): a 256 MiB write (2x the 126 MB L2) on the timing stream,
    issued outside each step's event bracket."""

    BYTES = 256 << 20

    def __init__(self):
        import torch

        self.buf = torch.empty(self.BYTES, dtype=torch.uint8, device="cuda")
        self.n = 0

    def __call__(self):
        self.n += 1
        self.buf.fill_(self.n & 0xFF)

    def note(self):
        return f"L2 flushed between timed steps ({self.BYTES >> 20} MiB write outside each step's events)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for name, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---- workload setup ---------------------------------------------------------------

class Workload:
    """Device-resident inputs of this rank's share of the workload."""

    def __init__(self, name: str, rank: int, world: int, scale: int, c1_mode: str = "shadow"):
        import torch

        from paper_1304_3771_b200 import dataplane as dp
        from paper_1304_3771_b200 import shard
        from paper_1304_3771_b200 import workloads as W

        self.name = name
        t0 = time.time()
        if name == "c5":
            cfg = W.C5Config() if scale == 1 else W.C5Config().scaled(scale)
            self.cfg = cfg
            owned = shard.owned_guests(cfg.guests, rank, world)
            self.owned = owned
            # a rank of an N-rank job holds the host-private region + its own guests' slots in HBM
            # (pv_image_create); one rank holds everything
            wd = W.build_c5(cfg, device=True, resident_guests=owned if world > 1 else None)
            self.world = wd
            self.memv = wd.memv
            t_spaces, bounds, vas_parts, self.proc_vas = [], [], [], []
            self.proc_lane0 = []  # global lane offset of every (guest, process) batch: guest order, then process
            lane = 0
            for g in owned:
                g0 = g * cfg.vas_per_guest
                for p, v in enumerate(W.c5_vas(cfg, g)):
                    t_spaces.append(W.c5_shadow_space(wd, g, p))
                    bounds.append((lane, lane + len(v), len(t_spaces) - 1))
                    vas_parts.append(v)
                    self.proc_vas.append((g, p, v))
                    self.proc_lane0.append(g0)
                    g0 += len(v)
                    lane += len(v)
            self.n_vas = lane
            self.total_vas = cfg.guests * cfg.vas_per_guest
            c_spaces, c_shims, rows = [], [], []
            self.proc_ops = []
            buf_off = 0
            for g in owned:
                for p, ops in enumerate(W.c5_ops(cfg, g)):
                    c_spaces.append(W.c5_hybrid_space(wd, g, p))
                    c_shims.append(W.c5_shim(wd, g, p))
                    si = len(c_spaces) - 1
                    offs = buf_off + np.arange(len(ops), dtype=np.uint64) * np.uint64(cfg.op_bytes)
                    rows.append(np.stack([ops[:, 0], ops[:, 1], offs, np.full(len(ops), si, np.uint64)], 1))
                    self.proc_ops.append((g, p, ops, offs))
                    buf_off += int(ops[:, 1].sum())
            self.copy_bytes = buf_off
            self.total_copy_bytes = cfg.guests * cfg.copy_bytes_per_guest
            ops_all = np.concatenate(rows)
        elif c1_mode == "4l":
            # BASELINE configs[0] as written: a 4-level 4 KiB table (extension geometry, parity pinned
            # by the C restatement orc_walk4 only); no e2e / CPU arm (no reference API for it)
            from paper_1304_3771_b200 import ext4l as X

            mem, t4 = X.build_c1_4l()
            self.c1_mode = c1_mode
            self.memv = None
            self.image_mem = mem
            self.owned = [0]
            t_spaces = [t4.space]
            v_all = X.c1_4l_vas()
            lo, hi = len(v_all) * rank // world, len(v_all) * (rank + 1) // world
            v = v_all[lo:hi]
            vas_parts = [v]
            bounds = [(0, len(v), 0)]
            self.n_vas, self.total_vas = len(v), len(v_all)
            self.proc_vas, self.proc_lane0 = [(0, 0, v)], [lo]
            c_spaces, c_shims = [t4.space], None
            total = 64 << 20
            pages = total // 4096
            p0, p1 = pages * rank // world, pages * (rank + 1) // world
            n = (p1 - p0) * 4096
            ops_all = np.array([[X.C1_4L_VA + p0 * 4096, n, 0, 0]], dtype=np.uint64)
            self.proc_ops = [(0, 0, ops_all[:, :2], np.zeros(1, np.uint64))]
            self.copy_bytes, self.total_copy_bytes = n, total
            self.c1_space = None
        else:
            memv, guest, space = W.build_c1(c1_mode)
            self.c1_mode = c1_mode
            self.memv = memv
            self.owned = [0]
            tr = memv.translator(space, use_cache=False)
            t_spaces = [tr.device_space]
            v_all = W.c1_vas().astype(np.uint32)
            # one guest, one process: the VA range splits evenly over the ranks (the
            # image is replicated, walks are read-only) and the 64 MiB copy_to_user into page-aligned,
            # disjoint destination ranges, each written by exactly one rank
            lo, hi = len(v_all) * rank // world, len(v_all) * (rank + 1) // world
            v = v_all[lo:hi]
            vas_parts = [v]
            bounds = [(0, len(v), 0)]
            self.n_vas = len(v)
            self.total_vas = len(v_all)
            self.proc_vas = [(0, 0, v)]
            self.proc_lane0 = [lo]
            c_spaces = [tr.device_space]
            c_shims = None
            total = 64 << 20
            pages = total // 4096
            p0, p1 = pages * rank // world, pages * (rank + 1) // world
            n = (p1 - p0) * 4096
            ops_all = np.array([[W.C1_GVA + p0 * 4096, n, 0, 0]], dtype=np.uint64)
            self.proc_ops = [(0, 0, ops_all[:, :2], np.zeros(1, np.uint64))]
            self.copy_bytes = n
            self.total_copy_bytes = total
            self.c1_space = space
        self.build_s = time.time() - t0
        self.image = self.memv.host_mem.backing if self.memv is not None else self.image_mem.backing
        self.image.device()  # allocate + push tables
        allv = np.concatenate(vas_parts)
        self.vas = torch.from_numpy(allv.view(np.int32 if allv.dtype == np.uint32 else np.int64)).to("cuda")
        self.tplan = dp.TranslatePlan(t_spaces, bounds)
        self.t_spaces, self.t_bounds, self.c_spaces = t_spaces, bounds, c_spaces
        n = self.n_vas
        self.out = (torch.empty(n, dtype=torch.int64, device="cuda"), torch.empty(n, dtype=torch.int32, device="cuda"),
                    torch.zeros(n, dtype=torch.int64, device="cuda"))
        self.cplan = dp.CopyPlan(c_spaces, ops_all, shims=c_shims)
        g = torch.Generator(device="cuda")
        g.manual_seed(1304 + rank)
        self.src = torch.randint(0, 256, (max(self.copy_bytes, 1),), dtype=torch.uint8, device="cuda", generator=g)
        torch.cuda.synchronize()


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as tdist

    from paper_1304_3771_b200 import _native as N
    from paper_1304_3771_b200 import dataplane as dp
    from paper_1304_3771_b200 import shard

    torch.cuda.set_device(local)
    wl = Workload(args.workload, rank, world, args.scale, args.c1_mode)
    lib = N.lib()
    img = wl.image
    dev = img.device()
    plan = wl.cplan
    stream = torch.cuda.current_stream()
    s = stream.cuda_stream
    owner = dp._owner_map(img)
    shim_scratch = dp._shim_scratch(img, plan.n_pages) if plan.shims is not None else None
    hint = dp.exec_hint(plan, wl.src.data_ptr())

    form = args.walk_form
    if form == "words":  # one 4-byte word per lane + exception records (pv_translate_words)
        w_words = torch.empty(wl.n_vas, dtype=torch.int32, device="cuda")
        w_exc = dp.ExcList(min(wl.n_vas, 1 << 20))

    # C5 at N > 1: every rank's walk stores its lane words straight into rank 0's HBM (one buffer, rank-major
    # sections) -- the result return fused into the walk over NVLink / NVSwitch peer memory
    peer, peer_off, peer_note = None, 0, None
    if form == "words" and wl.name == "c5" and world > 1 and _pg() and not args.no_peer_return:
        counts = [None] * world
        tdist.all_gather_object(counts, int(wl.n_vas))
        peer_off = sum(counts[:rank])
        try:
            peer = shard.PeerResultBuffer(4 * sum(counts), rank, world)
        except Exception as exc:  # noqa: BLE001 - no peer mapping: local output + the separate gather
            peer_note = f"peer mapping unavailable ({type(exc).__name__}: {str(exc)[:100]})"
    w_out = (peer.ptr + 4 * peer_off) if peer is not None else (w_words if form == "words" else None)

    def phase_translate():
        if form == "words":
            w_exc.reset()
            dp.translate_words(img, wl.tplan, wl.vas, w_out, w_exc)
        elif form == "packed":  # PV_OUT_PACKED: one u64 per lane, no status array
            dp.translate_lanes(img, wl.tplan, wl.vas, out=(wl.out[0], None, wl.out[2]), packed=True)
        else:
            dp.translate_lanes(img, wl.tplan, wl.vas, out=wl.out)

    def phase_translate_conc():  # the same walk sized to share every SM with the exec (PV_CONCURRENT)
        if form == "words":
            w_exc.reset()
            dp.translate_words(img, wl.tplan, wl.vas, w_out, w_exc, concurrent=True)
        elif form == "packed":
            dp.translate_lanes(img, wl.tplan, wl.vas, out=(wl.out[0], None, wl.out[2]), packed=True, concurrent=True)
        else:
            dp.translate_lanes(img, wl.tplan, wl.vas, out=wl.out, concurrent=True)

    def phase_plan():  # fills + plan + trap shim + conflict stamp
        cs = torch.cuda.current_stream().cuda_stream
        plan.first_bad.fill_(-1)
        plan.results.zero_()
        plan.conflict.zero_()
        # a captured step keeps this epoch: its stamps (epoch, chunk) and table-node marks repeat
        # identically, never a conflict
        epoch = owner.next_epoch()
        N.check(lib.pv_copy_plan_nodes(dev.data_ptr(), img.nbytes, plan.spaces.data_ptr(), plan.ops.data_ptr(),
                                       plan.n_ops, plan.page_off.data_ptr(), plan.n_pages,
                                       plan.page_hpa.data_ptr(), plan.page_status.data_ptr(),
                                       plan.page_aux.data_ptr(), plan.first_bad.data_ptr(), owner.nodes.data_ptr(),
                                       owner.npages, epoch, cs), "plan")
        if plan.shims is not None:  # the hybrid resolver's trap shim (none trap in C5: empty passes)
            N.check(lib.pv_copy_shim(dev.data_ptr(), img.nbytes, plan.spaces.data_ptr(), plan.shims.data_ptr(),
                                     plan.ops.data_ptr(), plan.n_ops, plan.page_off.data_ptr(), plan.n_pages,
                                     plan.page_hpa.data_ptr(), plan.page_status.data_ptr(), plan.first_bad.data_ptr(),
                                     img.dirty_map().data_ptr(), plan.shim_written.data_ptr(), shim_scratch.data_ptr(),
                                     shim_scratch.numel(), cs), "shim")
        N.check(lib.pv_copy_stamp(plan.page_off.data_ptr(), plan.n_ops, plan.n_pages, plan.page_hpa.data_ptr(),
                                  plan.first_bad.data_ptr(), owner.map.data_ptr(), img.npages, epoch,
                                  plan.conflict.data_ptr(), owner.nodes.data_ptr(), cs), "stamp")

    def phase_exec():
        cs = torch.cuda.current_stream().cuda_stream
        N.check(lib.pv_copy_exec(dev.data_ptr(), img.nbytes, plan.ops.data_ptr(), plan.n_ops,
                                 plan.page_off.data_ptr(), plan.n_pages, N.TO_GUEST | hint, plan.page_hpa.data_ptr(),
                                 plan.page_status.data_ptr(), plan.page_aux.data_ptr(), plan.first_bad.data_ptr(),
                                 wl.src.data_ptr(), wl.src.numel(), plan.results.data_ptr(),
                                 img.dirty_map().data_ptr(), plan.conflict.data_ptr(), cs), "exec")

    graphs = None

    def step(ev):
        ev[0].record(stream)
        if graphs:
            graphs[0].replay()
        else:
            phase_translate()
        ev[1].record(stream)
        ev[2].record(stream)
        if graphs:
            graphs[1].replay()
        else:
            phase_plan()
        ev[3].record(stream)
        if graphs:
            graphs[2].replay()
        else:
            phase_exec()
        ev[4].record(stream)
        img.note_device_write()

    side = torch.cuda.Stream()

    def step_overlap(ev):
        """One step with the walk on a second stream beside plan + exec: the
        walk is bound by the SM->L2 request port, the exec by HBM bandwidth,
        and they are independent (different guests' requests; the batch
        writes no table page -- the stamp pass's table-hazard check)."""
        ev[0].record(stream)
        side.wait_event(ev[0])
        with torch.cuda.stream(side):
            graphs[3].replay() if graphs else phase_translate_conc()
            ev[2].record(side)
        graphs[1].replay() if graphs else phase_plan()
        graphs[2].replay() if graphs else phase_exec()
        stream.wait_event(ev[2])
        ev[1].record(stream)
        img.note_device_write()

    split, split_note, split_cands, split_tune = None, None, [], None
    split_sms = args.split_sms if args.split_sms is not None else (64 if wl.name == "c5" else 0)
    if split_sms and not args.overlap:
        try:
            # the placement of the two SM sets over the GPCs (the driver's co-scheduled 8-SM groups, single-SM
            # granularity, either one interleaved) changes the step by a few %, and which is fastest depends on
            # the box: all are timed before the timed region and the fastest is kept
            split_cands = [dp.SmSplit(split_sms)]
            for fine, inter in ((True, False), (False, True), (True, True)):
                try:
                    split_cands.append(dp.SmSplit(split_sms, fine=fine, interleave=inter))
                except Exception:  # noqa: BLE001 - a placement the driver refuses is skipped
                    pass
            split = split_cands[0]
        except Exception as exc:  # noqa: BLE001 - no green contexts: the phases run back to back
            split_note = f"SM split unavailable ({type(exc).__name__}: {str(exc)[:100]}): phases back to back"

    def step_split(ev):
        """One step with the walk on SM partition 0 beside plan + exec on
        partition 1 (disjoint SMs; the batch writes no table page -- the
        stamp pass's table-hazard check -- so the walk reads the same tables
        either way)."""
        ev[0].record(stream)
        for k in (0, 1):
            split.streams[k].wait_event(ev[0])
        with split.on(0) as sa:
            phase_translate()
            ev[2].record(sa)
        with split.on(1) as sb:
            ev[3].record(sb)
            phase_plan()
            ev[4].record(sb)
            phase_exec()
            ev[5].record(sb)
        stream.wait_event(ev[2])
        stream.wait_event(ev[5])
        ev[1].record(stream)
        img.note_device_write()

    def barrier():
        if world > 1 and tdist.is_initialized():
            tdist.barrier()

    for _ in range(args.warmup):
        step([torch.cuda.Event(enable_timing=True) for _ in range(5)])
        if split is not None:
            step_split([torch.cuda.Event(enable_timing=True) for _ in range(6)])
    torch.cuda.synchronize()
    launch_mode = "eager"
    if not args.no_graph:
        # CUDA graphs of the three phases (the kernels and their arguments are identical every step),
        # replayed between the per-phase events: no per-launch host/driver gaps inside a phase
        try:
            gs = [torch.cuda.CUDAGraph() for _ in range(4)]
            for g, fn in zip(gs, (phase_translate, phase_plan, phase_exec, phase_translate_conc)):
                with torch.cuda.graph(g):
                    fn()
            img.note_device_write()
            torch.cuda.synchronize()
            graphs = gs
            for _ in range(2):
                step([torch.cuda.Event(enable_timing=True) for _ in range(5)])
                step_overlap([torch.cuda.Event(enable_timing=True) for _ in range(3)])
            torch.cuda.synchronize()
            launch_mode = "cuda_graph"
        except Exception as exc:  # noqa: BLE001 - eager launches are the same kernels
            graphs = None
            launch_mode = f"eager (graph capture failed: {type(exc).__name__}: {str(exc)[:120]})"
            torch.cuda.synchronize()

    if len(split_cands) > 1:
        split_tune = {}
        for cand in split_cands:
            split = cand
            for _ in range(2):
                step_split([torch.cuda.Event(enable_timing=True) for _ in range(6)])
            torch.cuda.synchronize()
            t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0e.record(stream)
            for _ in range(5):
                step_split([torch.cuda.Event(enable_timing=True) for _ in range(6)])
            t1e.record(stream)
            torch.cuda.synchronize()
            split_tune[cand.placement] = t0e.elapsed_time(t1e) / 5
        times = shard.max_over_ranks([split_tune[c.placement] for c in split_cands], world, device="cuda")
        split = split_cands[min(range(len(split_cands)), key=lambda k: times[k])]  # every rank: the same choice
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    overlap = args.overlap or split is not None
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    ovs = [[torch.cuda.Event(enable_timing=True) for _ in range(6 if split is not None else 3)]
           for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    # C1's inputs fit in L2: flush it between steps, outside each step's bracket
    flush = L2Flush() if wl.name != "c5" else None
    brackets = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
    # the timed region: K steps (walk beside plan + exec unless --serial-step)
    barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for k in range(args.steps):
        if flush is not None:
            flush()
        brackets[k][0].record(stream)
        if split is not None:
            step_split(ovs[k])
        elif overlap:
            step_overlap(ovs[k])
        else:
            step(evs[k])
        brackets[k][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier()
    total_ms = (t_start.elapsed_time(t_end) if flush is None
                else sum(a.elapsed_time(b) for a, b in brackets))
    split_out = None
    if split is not None:  # the split steps' lane results, compared with the serial steps' below
        split_out = (w_words if form == "words" else wl.out[0]).clone()
    if overlap:
        # per-phase figures (value, rooflines): K more steps with the phases back to back
        barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            if flush is not None:
                flush()
            step(evs[k])
        torch.cuda.synchronize()
        barrier()
    peer_return = None
    if peer is not None:
        # this rank's words, read back from rank 0's memory: what the checks below decode; rank 0 checks that
        # its buffer holds every rank's section as that rank computed it
        peer.copy_out(w_words.data_ptr(), 4 * peer_off, 4 * wl.n_vas, stream.cuda_stream)
        torch.cuda.synchronize()
        mine = hashlib.sha256(w_words.cpu().numpy().tobytes()).hexdigest()
        sections = [None] * world
        tdist.all_gather_object(sections, (peer_off, int(wl.n_vas), mine))
        verified = None
        if rank == 0:
            full = torch.empty(sum(n for _, n, _ in sections), dtype=torch.int32, device="cuda")
            peer.copy_out(full.data_ptr(), 0, 4 * full.numel(), stream.cuda_stream)
            host = full.cpu().numpy()
            verified = all(hashlib.sha256(host[o:o + n].tobytes()).hexdigest() == d for o, n, d in sections)
        peer_return = {"mode": "peer stores fused into the walk: each rank's walk writes its lane words "
                               "straight into rank 0's HBM (CUDA IPC mapping, NVLink / NVSwitch)",
                       "bytes": 4 * sum(n for _, n, _ in sections),
                       "remote_bytes": 4 * sum(n for r, (_, n, _) in enumerate(sections) if r != 0),
                       "in_timed_region": True, "verified": verified}
    same_split = None
    if split_out is not None:
        same_split = bool(torch.equal(split_out, w_words if form == "words" else wl.out[0]))
    clk = clocks.stop()
    # correctness of the timed configuration: no conflicts, every op complete
    assert int(plan.conflict.item()) == 0, "conflicting destinations in the bench batch"
    res = plan.results.cpu().numpy().view(np.uint64)
    assert (res[:, 3] & 0xFFFFFFFF == 0).all() and (res[:, 0] == plan.host_ops[:, 1]).all()
    other = None
    n_exc = None
    if form != "unpacked":  # decode the timed step's lane words for the checks below
        if form == "words":
            exc, n_exc, overflow = w_exc.read()
            assert not overflow, "more exception lanes than the bench's record list holds"
            v, st_, _ = dp.unpack_words(w_words.cpu().numpy(), wl.vas.cpu().numpy(), exc)
        else:
            v, st_ = dp.unpack_lanes(wl.out[0].cpu().numpy(), wl.out[2].cpu().numpy())
        wl.out[0].copy_(torch.from_numpy(v.view(np.int64)))
        wl.out[1].copy_(torch.from_numpy(st_.view(np.int32)))
        # A/B in the same run: the walk in the next wider form, K launches, same lanes and results
        o2 = (torch.empty_like(wl.out[0]), torch.empty_like(wl.out[1]), torch.zeros_like(wl.out[2]))
        wide = form == "words"  # words -> PV_OUT_PACKED u64; packed -> (value, status)

        def other_walk():
            if wide:
                dp.translate_lanes(img, wl.tplan, wl.vas, out=(o2[0], None, o2[2]), packed=True)
            else:
                dp.translate_lanes(img, wl.tplan, wl.vas, out=o2)
        other_walk()
        o_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
        for a, b in o_ev:
            if flush is not None:
                flush()
            a.record(stream)
            other_walk()
            b.record(stream)
        torch.cuda.synchronize()
        if wide:
            ov, os_ = dp.unpack_lanes(o2[0].cpu().numpy(), o2[2].cpu().numpy())
            same = bool(np.array_equal(ov, v) and np.array_equal(os_, st_))
        else:
            same = bool(torch.equal(o2[0], wl.out[0]) and torch.equal(o2[1], wl.out[1]))
        other = {"form": "PV_OUT_PACKED (one u64 per lane)" if wide else "unpacked (u64 value + u32 status)",
                 "translate_ms_per_step": sum(a.elapsed_time(b) for a, b in o_ev) / args.steps, "launch": "eager",
                 "results_equal": same}
    n_faults = int((wl.out[1] != 0).sum().item())
    tr_ms = sum(e[0].elapsed_time(e[1]) for e in evs)
    serial_ms = sum(e[0].elapsed_time(e[4]) for e in evs)
    ov_walk_ms = sum(e[0].elapsed_time(e[2]) for e in ovs) if overlap else None
    split_phases = None
    if split is not None:
        split_phases = {"sms": {"walk": split.sms[0], "plan_exec": split.sms[1]},
                        "placement": split.placement,
                        "tuned_ms_per_step": split_tune,
                        "walk_ms": sum(e[0].elapsed_time(e[2]) for e in ovs) / args.steps,
                        "plan_ms": sum(e[3].elapsed_time(e[4]) for e in ovs) / args.steps,
                        "exec_ms": sum(e[4].elapsed_time(e[5]) for e in ovs) / args.steps,
                        "lanes_equal_serial_step": same_split}
    plan_ms = sum(e[2].elapsed_time(e[3]) for e in evs)
    exec_ms = sum(e[3].elapsed_time(e[4]) for e in evs)
    copy_ms = sum(e[1].elapsed_time(e[4]) for e in evs)
    # this rank's per-step spread (best and median of the timed steps)
    tr_steps = sorted(e[0].elapsed_time(e[1]) for e in evs)
    ex_steps = sorted(e[3].elapsed_time(e[4]) for e in evs)
    spread = {"translate_ms": {"best": tr_steps[0], "median": statistics.median(tr_steps)},
              "exec_ms": {"best": ex_steps[0], "median": statistics.median(ex_steps)}, "rank": rank}
    from paper_1304_3771_b200 import shard

    total_ms, tr_ms, copy_ms, exec_ms, plan_ms, serial_ms = shard.max_over_ranks(
        [total_ms, tr_ms, copy_ms, exec_ms, plan_ms, serial_ms], world, device="cuda")
    parity = None
    if not args.no_parity:
        parity = verify_parity(wl, cpu_threads())
    want_gather = (args.gather or (world > 1 and _pg() and peer is None)) and not args.no_gather
    gather = gather_results(wl, rank, world) if (want_gather and wl.name == "c5") else None
    K = args.steps
    trans_per_s = wl.total_vas * K / (tr_ms / 1e3) if world > 0 else 0.0
    copy_gbs = wl.total_copy_bytes * K / (copy_ms / 1e3) / 1e9

    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e and wl.memv is not None:
        try:
            e2e = run_e2e(wl, args, world)
        except Exception as exc:  # noqa: BLE001 - reported in the line (the device figures stand)
            if world > 1:
                raise  # ranks must not diverge on collectives
            e2e = {"error": f"{type(exc).__name__}: {str(exc)[:300]}"}

    peak, peak_kind = peaks()
    exec_achieved = 2 * wl.copy_bytes * K / (exec_ms / 1e3) / 1e9
    # u32 VA in + (u32 word | u64 lane word | u64 hpa + u32 status) out
    walk_bytes = {"words": 8, "packed": 12, "unpacked": 16}[form] * wl.n_vas
    walk_achieved = walk_bytes * K / (tr_ms / 1e3) / 1e9
    walk_bytes_pte = walk_bytes + 8 * _leaf_ptes(wl)  # + 8 B per distinct leaf PTE
    walk_achieved_pte = walk_bytes_pte * K / (tr_ms / 1e3) / 1e9
    traffic = load_traffic(args.workload)
    line = {
        "metric": METRIC,
        "value": trans_per_s,
        "unit": "translations/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": total_ms / K,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u64 (integer walk) / u8 (payload)",
        "data": "synthetic",
        "config": config_of(wl, world),
        "copy": {"value": copy_gbs, "unit": "GB/s", "payload_bytes_per_step": wl.total_copy_bytes,
                 "ms_per_step": copy_ms / K, "exec_ms_per_step": exec_ms / K,
                 "plan_shim_stamp_ms_per_step": plan_ms / K},
        "translate_ms_per_step": tr_ms / K,
        "walk_form": {"words": "pv_translate_words (one u32 per lane + exception records)",
                      "packed": "PV_OUT_PACKED (one u64 per lane)",
                      "unpacked": "unpacked (u64 value + u32 status)"}[form],
        "exception_records": n_exc,
        "walk_other_form": other,
        "step": {"mode": ("split" if split is not None else "overlapped") if overlap else "serial",
                 "split": split_phases, "split_note": split_note,
                 "ms": total_ms / K, "serial_ms": serial_ms / K,
                 "translations_per_s": wl.total_vas * K / (total_ms / 1e3),
                 "copy_gbs": wl.total_copy_bytes * K / (total_ms / 1e3) / 1e9,
                 "walk_ms_in_overlap": None if ov_walk_ms is None else ov_walk_ms / K,
                 "hbm_floor_ms": (2 * wl.copy_bytes + walk_bytes + 8 * _leaf_ptes(wl)) / (peak * 1e6),
                 "note": ("ms_per_step = one step with the walk on its own SM partition (green context, "
                          "pv_sm_split) beside plan + exec on the rest; both read/write HBM at once, so each runs "
                          "slower than alone but the step is shorter than back to back (serial_ms); value, copy "
                          "and the rooflines come from K more steps with the phases back to back, and the split "
                          "step's lane results equal theirs (split.lanes_equal_serial_step)")
                 if split is not None else
                 ("ms_per_step = one step with the walk on a second stream beside plan + exec "
                  "(PV_CONCURRENT: one walker CTA per SM next to the exec's); value, copy and the "
                  "rooflines come from K more steps with the phases back to back (serial_ms)")
                 if overlap else ("phases back to back (--split-sms N puts the walk on its own SM partition "
                                  "beside plan + exec)")},
        "per_step": spread,
        "roofline": {"bound": "hbm",
                     "kernel": "pv_copy_exec (" + ("exec_bulk_kernel, TMA" if hint else "exec_kernel, LSU") + ")",
                     "achieved": exec_achieved,
                     "peak": peak, "unit": "GB/s", "frac": exec_achieved / peak, "peak_source": peak_kind,
                     "traffic": traffic_for(traffic, "exec", 2 * wl.copy_bytes),
                     "frac_of_8tbs_spec": exec_achieved / 8000.0,
                     "algorithmic_bytes_per_launch": 2 * wl.copy_bytes},
        "roofline_walk": {"bound": "hbm", "kernel": "pv_translate (translate_kernel)", "achieved": walk_achieved,
                          "peak": peak, "unit": "GB/s", "frac": walk_achieved / peak,
                          "traffic": traffic_for(traffic, "translate", walk_bytes),
                          "algorithmic_bytes_per_launch": walk_bytes,
                          "with_leaf_ptes": {"algorithmic_bytes_per_launch": walk_bytes_pte,
                                             "distinct_leaf_ptes": _leaf_ptes(wl), "achieved": walk_achieved_pte,
                                             "frac": walk_achieved_pte / peak},
                          "note": {"words": "8 B/translation (u32 VA in, one u32 lane word out)",
                                   "packed": "12 B/translation (u32 VA in, one u64 lane word out)",
                                   "unpacked": "16 B/translation (u32 VA in, u64 hpa + u32 status out)"}[form]
                                  + "; with_leaf_ptes adds "
                                  "SURVEY.md 8(d)'s 8 B per distinct leaf PTE touched",
                          "gather_sol": walker_sol(wl.n_vas * K / (tr_ms / 1e3), form),
                          "ncu": load_json_profile("walker_ncu.json")},
        "faulting_lanes": n_faults,
        "parity": parity,
        "gather_to_rank0": gather,
        "results_to_rank0": peer_return if peer is not None else peer_note,
        "hbm_image": {"image_bytes": img.nbytes, "device_bytes": img.device_bytes,
                      "resident": "all" if not img.partial else
                      "host-private region + owned guests' slots (pv_image_create) + one shared hole"},
        "gpu_launches": (4 + (1 if wl.n_vas >= 8 * 296 * 2048 else 0) + 1
                         + (2 if wl.cplan.shims is not None else 0)) * K,
        "launch": launch_mode,
        "gpu_launches_note": "per step: stage-table pre-pass (batches of >= 8 chunks per CTA), translate, "
                             "leaf-index re-encode of pages the previous step's copies dirtied, plan, stamp, "
                             "exec (TMA bulk path), + the hybrid trap shim (eval + one cooperative resolve kernel "
                             "that returns at once when nothing traps); 3 torch fills not counted",
        "clocks": clk,
        "e2e": e2e,
        "build_s": wl.build_s,
        "provenance": provenance(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and wl.memv is not None:
        try:
            line["cpu_baseline"] = cpu_baseline(wl, args)
        except Exception as exc:  # noqa: BLE001 - reported in the line (the device figures stand)
            line["cpu_baseline"] = {"error": f"{type(exc).__name__}: {str(exc)[:300]}"}
    if peer is not None:
        peer.close()
    return line


def _leaf_ptes(wl) -> int:
    """Distinct leaf PTEs the walk reads (+ 8 B each): one per
    distinct (process, page) among the batch's VAs."""
    n = getattr(wl, "_leaf_ptes", None)
    if n is None:
        n = sum(len(np.unique(np.asarray(v) >> 12)) for _, _, v in wl.proc_vas)
        wl._leaf_ptes = n
    return n


def verify_parity(wl, threads: int, n_ops: int = 64) -> dict:
    """Full-size parity of the timed configuration (after the timed steps),
    against the C oracle (oracle/pvoracle.c -- test infrastructure, used here
    only as the checker):

    * every lane of the translate batch (value + status) equals
      ``O.translate`` of the same VA over the same tables;
    * ``n_ops`` copy ops spread over the batch: the destination bytes in HBM,
      at the pages the ORACLE translates the op's VAs to, equal the op's
      source bytes (copy_user_buffer semantics, memvirt.py:604-628).

    The oracle walks a host copy of the device image: the whole image when it
    is small, else the host-private region (every node of the C5 shadow and
    hybrid tables lives there; data pages are never read by a walk)."""
    import torch

    from oracle import oracle as O
    from paper_1304_3771_b200 import _native as N
    from paper_1304_3771_b200 import image as I

    t0 = time.perf_counter()
    img = wl.image
    dev = img.device()
    torch.cuda.synchronize()
    span = img.nbytes if img.nbytes <= (4 << 30) else wl.cfg.host_private
    if span < img.nbytes and any(sp.mode != N.ONE_STAGE for sp in wl.t_spaces + wl.c_spaces):
        raise RuntimeError("private-region parity needs one-stage (shadow / hybrid) spaces")
    ref = I._zeroed_host(img.nbytes)
    step = 256 << 20
    for a in range(0, span, step):
        ref[a:min(a + step, span)] = dev[a:min(a + step, span)].cpu().numpy()
    value = wl.out[0].cpu().numpy().view(np.uint64)
    status = wl.out[1].cpu().numpy().view(np.uint32)
    vas = wl.vas.cpu().numpy().view(np.uint32 if wl.vas.dtype == torch.int32 else np.uint64)
    lane_bad = 0
    for begin, end, si in wl.t_bounds:
        sp = wl.t_spaces[si]
        v, st, _ = O.translate(ref, O.space(sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode),
                               vas[begin:end].astype(np.uint64), threads=threads)
        lane_bad += int(((v != value[begin:end]) | (st != status[begin:end])).sum())
    t_lanes = time.perf_counter() - t0
    # copy ops: evenly spaced sample
    ops = wl.cplan.host_ops
    pick = np.unique(np.linspace(0, len(ops) - 1, min(n_ops, len(ops))).astype(np.int64))
    lib = N.lib()
    s = torch.cuda.current_stream().cuda_stream
    byte_bad, bytes_checked = 0, 0
    for i in pick.tolist():
        gva, ln, off, si = (int(x) for x in ops[i])
        sp = wl.c_spaces[si]
        n_pg = ((gva + ln - 1) >> 12) - (gva >> 12) + 1
        page_vas = ((gva >> 12) + np.arange(n_pg, dtype=np.uint64)) << np.uint64(12)
        v, st, _ = O.translate(ref, O.space(sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode), page_vas,
                               want_pfn=True, threads=threads)
        if (st != 0).any():
            byte_bad += ln
            continue
        pfns = torch.from_numpy(v.astype(np.int64)).cuda()
        got = torch.empty(n_pg * 4096, dtype=torch.uint8, device="cuda")
        N.check(lib.pv_gather_pages(dev.data_ptr(), img.nbytes, pfns.data_ptr(), n_pg, got.data_ptr(), s),
                "pv_gather_pages")
        head = gva & 0xFFF
        byte_bad += int((got[head:head + ln] != wl.src[off:off + ln]).sum().item())
        bytes_checked += ln
    return {"lanes": int(len(vas)), "lane_mismatches": lane_bad, "ops_checked": int(len(pick)),
            "bytes_checked": bytes_checked, "byte_mismatches": byte_bad,
            "oracle": "oracle/pvoracle.c (O.translate over a host copy of the image, %d threads)" % threads,
            "seconds": round(time.perf_counter() - t0, 2), "lanes_seconds": round(t_lanes, 2),
            "ok": lane_bad == 0 and byte_bad == 0}


def gather_results(wl, rank, world):
    """Return each owned guest's translation results to rank 0 (timed
    separately from the step: it is result delivery, not the data plane)."""
    import torch

    from paper_1304_3771_b200 import shard

    cfg = wl.cfg
    value, status, _ = wl.out
    per_guest, lane = {}, 0
    for g in shard.owned_guests(cfg.guests, rank, world):
        n = cfg.vas_per_guest
        per_guest[g] = {"value": value[lane:lane + n], "status": status[lane:lane + n]}
        lane += n

    def like(g):
        return {"value": torch.empty(cfg.vas_per_guest, dtype=torch.int64, device="cuda"),
                "status": torch.empty(cfg.vas_per_guest, dtype=torch.int32, device="cuda")}

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    got = shard.gather_to_rank0(per_guest, cfg.guests, rank, world, like)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    (dt,) = shard.max_over_ranks([dt], world, device="cuda")
    nbytes = cfg.guests * cfg.vas_per_guest * 12
    ok = digest = None
    if rank == 0:
        ok = sorted(got) == list(range(cfg.guests))
        h = hashlib.sha256()
        for g in range(cfg.guests):  # every guest's results, in guest order (equal at any N)
            h.update(got[g]["value"].cpu().numpy().tobytes())
            h.update(got[g]["status"].cpu().numpy().tobytes())
        digest = h.hexdigest()
    return {"ms": dt * 1e3, "bytes": nbytes, "remote_bytes": nbytes * (world - 1) // world, "complete": ok,
            "digest": digest}


def c2_device_payload(lens: np.ndarray):
    """IOCTL_SNAPSHOT blobs (devices.py:162-166) back to back, built on the
    device in chunks: byte j of op i = (j * 7 + 3) & 0xFF."""
    import torch

    offs = np.zeros(len(lens), dtype=np.int64)
    if len(lens) > 1:
        np.cumsum(lens[:-1], out=offs[1:])
    total = int(lens.sum())
    buf = torch.empty(total, dtype=torch.uint8, device="cuda")
    step = 50_000
    for a in range(0, len(lens), step):
        ln = torch.from_numpy(lens[a:a + step]).cuda()
        start = int(offs[a])
        n = int(ln.sum())
        local = torch.arange(n, device="cuda", dtype=torch.int64)
        base = torch.repeat_interleave(torch.from_numpy(offs[a:a + step] - start).cuda(), ln)
        buf[start:start + n] = ((local - base) * 7 + 3).remainder(256).to(torch.uint8)
    return buf, offs


def run_c2(args, rank, world, local):
    """BASELINE config 2: a trace of IOCTL_SNAPSHOT ioctls forwarded to a TDP
    guest's 8 processes (software HAS, FIFO-cached translators); each op
    stages its driver blob into the caller's arena with copy_to_user
    (backend.py:526-534).  One step = the whole trace as one batch: plan
    (one 2-stage translation per page), exact parallel FIFO replay, conflict
    stamp, ordered last-writer-wins apply.  Processes shard over ranks."""
    import torch

    from paper_1304_3771_b200 import _native as N
    from paper_1304_3771_b200 import dataplane as dp
    from paper_1304_3771_b200 import memvirt as mv
    from paper_1304_3771_b200 import shard
    from paper_1304_3771_b200 import workloads as W

    torch.cuda.set_device(local)
    t0 = time.time()
    memv, guest, spaces = W.build_c2()
    procs, gvas, lens = W.c2_trace(args.c2_ops)
    mine = np.isin(procs, shard.owned_guests(len(spaces), rank, world))
    procs, gvas, lens = procs[mine], gvas[mine], lens[mine]
    buf, offs = c2_device_payload(lens)
    trs = [memv.translator(sp, mv.TranslationCache()) for sp in spaces]
    rows = np.stack([gvas, lens, offs, procs], 1).astype(np.uint64)
    groups = [np.flatnonzero(procs == p) for p in range(len(spaces))]
    groups = [g for g in groups]
    img = memv.host_mem.backing
    plan = dp.CopyPlan([t.device_space for t in trs], rows, fifo_groups=groups)
    fifo0 = dp.pack_fifo([t.cache for t in trs])
    fifo = dp._to_dev(fifo0)
    # the forwarding leg (frontend pack -> backend identify + reassemble,
    # hypercall.py:125-211): the trace as IOCTL FileOps, one vCPU per process
    from paper_1304_3771_b200 import hypercall as hc

    reg = hc.VcpuRegistry()
    for p, sp in enumerate(spaces):
        reg.register_vcpu(p, guest.guest_id)
        reg.register_process(guest.guest_id, sp.cr3, sp.pid)
    fops = np.zeros((len(gvas), N.FOP_WORDS), dtype=np.uint64)
    fops[:, 0] = int(hc.FileOpKind.IOCTL)
    fops[:, 1 + hc._FIELD_INDEX["handle"]] = 3
    fops[:, 1 + hc._FIELD_INDEX["cmd"]] = W.IOCTL_SNAPSHOT
    fops[:, 1 + hc._FIELD_INDEX["arg_gva"]] = gvas
    fops[:, 1 + hc._FIELD_INDEX["arg_len"]] = lens
    t64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()  # noqa: E731
    fops_d, vcpu_d = t64(fops), t64(procs)
    cr3_d = t64(np.array([spaces[p].cr3 for p in range(len(spaces))], dtype=np.uint64)[procs])
    tag_d = torch.zeros_like(vcpu_d)
    tables = reg.device_tables()
    fwd = {}
    build_s = time.time() - t0
    stream = torch.cuda.current_stream()

    def step(ev):
        ev[0].record(stream)
        frames, _, _ = hc.pack_device(fops_d, vcpu_d, cr3_d, tag_d, n_frames=len(gvas))
        fwd["ops"], fwd["status"], fwd["record"], _ = hc.dispatch_device(frames, reg, tables)
        ev[1].record(stream)
        graphs[0].replay() if graphs else phase_plan()
        ev[2].record(stream)
        graphs[1].replay() if graphs else phase_apply()
        ev[3].record(stream)
        img.note_device_write()

    def phase_plan():  # plan + exact FIFO replay + conflict stamp (+ the exec, which stands down)
        dp.copy_launch(img, plan, N.TO_GUEST, buf, fifo_dev=fifo, fifo_cap=10)

    def phase_apply():  # the ordered last-writer-wins path
        dp.copy_ordered(img, plan, buf)

    graphs = None
    for _ in range(args.warmup):
        step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
    torch.cuda.synchronize()
    launch_mode = "eager"
    if not args.no_graph:
        # the plan and apply phases as CUDA graphs (no host synchronisation inside them; the forwarding
        # leg stays eager: frame assembly reads its pairing-set size back)
        try:
            gs = [torch.cuda.CUDAGraph() for _ in range(2)]
            for g, fn in zip(gs, (phase_plan, phase_apply)):
                with torch.cuda.graph(g):
                    fn()
            img.note_device_write()
            torch.cuda.synchronize()
            graphs = gs
            for _ in range(2):
                step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
            torch.cuda.synchronize()
            launch_mode = "cuda_graph (plan + apply phases)"
        except Exception as exc:  # noqa: BLE001 - eager launches are the same kernels
            graphs = None
            launch_mode = f"eager (graph capture failed: {type(exc).__name__}: {str(exc)[:120]})"
            torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if world > 1 and _pg():
        import torch.distributed as tdist

        tdist.barrier()
    torch.cuda.synchronize()
    lib = N.lib()
    for k in range(args.steps):
        step(evs[k])
    torch.cuda.synchronize()
    clk = clocks.stop()
    # per-kernel launch times (rooflines, dominant kernel), from event-timed eager runs of the same phases
    lib.pv_timing(1)
    for _ in range(3):
        frames, _, _ = hc.pack_device(fops_d, vcpu_d, cr3_d, tag_d, n_frames=len(gvas))
        hc.dispatch_device(frames, reg, tables)
        phase_plan()
        phase_apply()
    torch.cuda.synchronize()
    n_apply = ctypes.c_uint64(0)
    kern_ms = lib.pv_timing_ms(b"ordered_apply", ctypes.byref(n_apply))
    kern_each = {}
    for name in C2_TIMED_KERNELS:
        n_l = ctypes.c_uint64(0)
        t = lib.pv_timing_ms(name.encode(), ctypes.byref(n_l))
        kern_each[name] = t / max(int(n_l.value), 1)
    lib.pv_timing(0)
    img.note_device_write()
    fwd_ms = sum(e[0].elapsed_time(e[1]) for e in evs)
    plan_ms = sum(e[1].elapsed_time(e[2]) for e in evs)
    apply_ms = sum(e[2].elapsed_time(e[3]) for e in evs)
    total_ms, fwd_ms, plan_ms, apply_ms, kern_ms = shard.max_over_ranks(
        [fwd_ms + plan_ms + apply_ms, fwd_ms, plan_ms, apply_ms, kern_ms], world, device="cuda")
    res = plan.results.cpu().numpy().view(np.uint64)
    assert (res[:, 3] & 0xFFFFFFFF == 0).all(), "C2 ops must all succeed"
    # the reassembled ops are the trace: arg_gva / arg_len / issuing process
    got = fwd["ops"].cpu().numpy().view(np.uint64)
    assert (fwd["status"].cpu().numpy() == 0).all()
    assert np.array_equal(got, fops)
    recs = tables[5]
    rec_pid = np.array([pid for _, pid in recs])[fwd["record"].cpu().numpy()]
    assert np.array_equal(rec_pid, np.array([sp.pid for sp in spaces])[procs])
    K = args.steps
    payload = int(W.c2_trace(args.c2_ops)[2].sum())
    peak, peak_kind = peaks()
    # algorithmic HBM bytes of one apply launch: only the bytes that survive
    # last-writer-wins have to move -- each distinct destination byte is read
    # once from its last writer's payload and written once.  (Per process the
    # ops' byte ranges are merged; processes write disjoint arenas.)
    surviving = 0
    for p in np.unique(procs).tolist():
        sel = procs == p
        a = np.sort(gvas[sel])
        order = np.argsort(gvas[sel], kind="stable")
        e = (gvas[sel] + lens[sel])[order]
        run_end = np.maximum.accumulate(e)
        starts = np.concatenate([[True], a[1:] > run_end[:-1]])
        idx = np.flatnonzero(starts)
        ends = np.concatenate([run_end[idx[1:] - 1], [run_end[-1]]])
        surviving += int((ends - a[idx]).sum())
    alg_bytes = 2 * surviving
    per_launch_ms = kern_ms / max(int(n_apply.value), 1)
    ach = alg_bytes / (per_launch_ms / 1e3) / 1e9
    kern_each = dict(zip(kern_each, shard.max_over_ranks(list(kern_each.values()), world, device="cuda")))
    kernels = c2_kernel_table(kern_each, len(gvas), plan.n_pages, per_launch_ms, alg_bytes, peak, peak_kind)
    dominant = max(kernels, key=lambda k: kernels[k]["launch_ms"])
    return {
        "metric": METRIC, "value": args.c2_ops * K / (total_ms / 1e3), "unit": "ioctls/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 (integer walk) / u8 (payload)", "data": "synthetic",
        "config": {"workload": f"C2: {args.c2_ops} IOCTL_SNAPSHOT ops forwarded as hypercall frames (frontend "
                               "pack, backend identify + reassemble) and their 64 B-4 KiB blobs staged by "
                               "copy_to_user into 8 processes' 1 MiB arenas of one TDP guest, software HAS (FIFO-10)",
                   "parallelism": f"process-sharded x{world}",
                   "l2": f"inputs larger than L2 ({args.c2_ops} x 136 B FileOp rows + 40 B frames, "
                         f"{payload / 1e9:.1f} GB of blobs per step)"},
        "copy": {"value": payload * K / (total_ms / 1e3) / 1e9, "unit": "GB/s (payload)"},
        "forward_ms_per_step": fwd_ms / K, "plan_fifo_ms_per_step": plan_ms / K,
        "ordered_apply_ms_per_step": apply_ms / K,
        "roofline": dict(kernels[dominant], kernel=dominant + "_kernel", dominant_by="event-timed launch ms "
                         "(pv_timing) among the step's kernels in `kernels`",
                         traffic=traffic_for(load_traffic("c2"), dominant, kernels[dominant]["alg_bytes_per_launch"])),
        "kernels": kernels,
        "payload_bytes_per_step": int(lens.sum()),
        "launch": launch_mode,
        "gpu_launches": 14 * K, "gpu_launches_note": "per step: frame pack, identify, classify, plan, 6 FIFO-replay "
                                                     "kernels (runs, spec, link, block, verify, apply), stamp, exec "
                                                     "(stands down), ordered keys (+ results), apply; CUB select / "
                                                     "radix sort / RLE / scan kernels not counted",
        "clocks": clk, "build_s": build_s,
        "cpu_baseline": (c2_cpu_baseline(memv, spaces, procs, gvas, lens, cpu_threads())
                         if rank == 0 and world == 1 and not args.no_cpu_baseline else None),
    }


C2_TIMED_KERNELS = ("frame_pack", "frame_classify", "plan", "fifo_spec", "stamp", "ordered_keys", "ordered_sort")


def c2_kernel_table(ms, n_ops, n_pages, apply_ms, apply_bytes, peak, peak_kind):
    """Per-kernel launch times of a C2 step (pv_timing event pairs) with the
    algorithmic HBM bytes each one must move and the
    resulting fraction of the measured HBM peak.  Sizes: FileOp row 136 B,
    frame 40 B, pv_op 32 B, pv_op_result 32 B, chunk descriptor 16 B."""
    alg = {  # kernel -> (bytes per launch, how they are counted)
        "frame_pack": (212 * n_ops, "per op: 136 B FileOp row + vcpu / cr3 / tag / frame slot (32 B) in, one 40 B "
                                    "frame + 4 B status out"),
        "frame_classify": (189 * n_ops, "per frame: 40 B frame + record + status in, 136 B op row + pair flag + "
                                        "iota out"),
        "plan": (48 * n_ops + 20 * n_pages, "per op: pv_op + page offset in, first-bad out; per page: hpa + status "
                                           "+ aux out (table nodes hit L2)"),
        "fifo_spec": (40 * n_ops + 44 * n_pages, "per FIFO-10 lookup: ref + op id + fresh hpa + status in, hit page "
                                                "+ flags out, window start / end states (~10.5 B per lookup); per "
                                                "op: pv_op + page offset.  Replays 32-lookup windows per warp (cache "
                                                "state in lanes, shuffles / match_any): bound by issue and dependent "
                                                "loads, not HBM"),
        "stamp": (16 * n_ops + 24 * n_pages, "per page: hpa in + owner word read-modify-write; per op: page offset "
                                             "+ first-bad"),
        "ordered_keys": (80 * n_ops + 32 * n_pages, "per op: pv_op + page offset + first-bad in, result out; per "
                                                    "page: hpa in, 4 B key + 16 B chunk descriptor + 4 B index out"),
        "ordered_sort": (36 * n_pages, "CUB onesweep radix sort of (4 B key, 4 B chunk index) pairs: a key "
                                       "histogram pass + two passes reading and writing every pair (the product "
                                       "build, PV_ORD_INDEX=1)"),
    }
    out = {}
    for k, t in ms.items():
        if t <= 0:
            continue
        b, note = alg[k]
        ach = b / (t / 1e3) / 1e9
        out[k] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                  "peak_source": peak_kind, "launch_ms": t, "alg_bytes_per_launch": b, "note": note}
    ach = apply_bytes / (apply_ms / 1e3) / 1e9
    out["ordered_apply"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                            "peak_source": peak_kind, "launch_ms": apply_ms, "alg_bytes_per_launch": apply_bytes,
                            "note": "bytes that survive last-writer-wins (each distinct destination byte read once "
                                    "from its last writer and written once); latency-bound (~2k destination pages, "
                                    "a few dependent TMA loads each)"}
    return out


def run_c3(args, rank, world, local):
    """BASELINE config 3 (extension geometry, parity unpinned by the
    reference): 16 GiB of device memory mmapped with alternating 2 MiB and
    4 KiB leaves under a 4-level table; one step = the sequential (4 KiB
    stride, 4,194,304 VAs) and strided (2 MiB + 4 KiB) batches."""
    import torch

    from paper_1304_3771_b200 import dataplane as dp
    from paper_1304_3771_b200 import ext4l as X
    from paper_1304_3771_b200 import shard

    torch.cuda.set_device(local)
    t0 = time.time()
    mem, t = X.build_c3()
    vas_h = np.concatenate([X.c3_sequential(), X.c3_strided()])
    vas_h = vas_h[rank::world]
    vas = torch.tensor(vas_h.view(np.int64), device="cuda")
    plan = dp.TranslatePlan([t.space], [(0, len(vas_h), 0)])
    out = (torch.empty(len(vas_h), dtype=torch.int64, device="cuda"),
           torch.empty(len(vas_h), dtype=torch.int32, device="cuda"),
           torch.zeros(len(vas_h), dtype=torch.int64, device="cuda"))
    mem.backing.device()
    build_s = time.time() - t0
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        dp.translate_lanes(mem.backing, plan, vas, out=out)
    torch.cuda.synchronize()
    graph, launch_mode = None, "eager"
    if not args.no_graph:  # one launch per step, replayed without host gaps
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                dp.translate_lanes(mem.backing, plan, vas, out=out)
            graph.replay()
            torch.cuda.synchronize()
            launch_mode = "cuda_graph"
        except Exception as exc:  # noqa: BLE001 - eager launches are the same kernel
            graph = None
            launch_mode = f"eager (graph capture failed: {type(exc).__name__}: {str(exc)[:120]})"
            torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    flush = L2Flush()  # 84 MB of lanes per step fit in L2: flushed between steps, outside the events
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for e0, e1 in evs:
        flush()
        e0.record(stream)
        graph.replay() if graph else dp.translate_lanes(mem.backing, plan, vas, out=out)
        e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    assert int((out[1] != 0).sum().item()) == 0
    (ms,) = shard.max_over_ranks([sum(a.elapsed_time(b) for a, b in evs)], world, device="cuda")
    total = len(X.c3_sequential()) + len(X.c3_strided())
    peak, peak_kind = peaks()
    ach = 20 * len(vas_h) * args.steps / (ms / 1e3) / 1e9
    return {
        "metric": METRIC, "value": total * args.steps / (ms / 1e3), "unit": "translations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 (integer walk)", "data": "synthetic",
        "config": {"workload": "C3 (extension geometry, parity unpinned): 16 GiB device mmap, alternating "
                               "2 MiB / 4 KiB leaves, 4-level 9/9/9/9/12 tables; sequential 4 KiB-stride + "
                               "strided 2 MiB+4 KiB batches", "lanes": total, "l2": flush.note()},
        "roofline": {"bound": "hbm", "kernel": "translate_generic_kernel", "achieved": ach, "peak": peak,
                     "unit": "GB/s", "frac": ach / peak, "peak_source": peak_kind,
                     "note": "20 B/translation (u64 VA in, u64 hpa + u32 status out)"},
        "launch": launch_mode, "gpu_launches": args.steps, "clocks": clk, "build_s": build_s,
        "cpu_baseline": (translate_cpu_baseline(mem.backing.host_for_read(), [t.space.s1_base, t.space.s1_root_pfn, 0,
                                                                              t.space.mode], vas_h,
                                                "4-level walks over the 16 GiB mixed-page mapping")
                         if rank == 0 and world == 1 and not args.no_cpu_baseline else None),
    }


def run_c4(args, rank, world, local):
    """BASELINE config 4 (fault-heavy): the C1 world with 20 % of the shadow
    leaves not present and 10 % trapping.  One step = 1 M translations
    (90 % in the region, 10 % uniform over 2^32: faults at every level,
    traps, bit-exact codes) through the shadow translator + a batch of 4096
    copy_to_user ops of 16 KiB through the hybrid resolver, whose trap shim
    runs on the device (pv_copy_shim fixes ~1,600 trapping slots per step).
    The trapping words are put back between steps, outside the timed region,
    so every step sees the same faults.  Lanes shard over ranks."""
    import random

    import torch

    from paper_1304_3771_b200 import _native as N
    from paper_1304_3771_b200 import dataplane as dp
    from paper_1304_3771_b200 import has
    from paper_1304_3771_b200 import shard
    from paper_1304_3771_b200 import workloads as W

    torch.cuda.set_device(local)
    t0 = time.time()
    memv, guest, space = W.build_c1("shadow", device=True)
    W.corrupt_c4(memv, space, "shadow")
    rec = has.GuestProcessRecord(_FakeGuest(0), space, memv)
    acc = has.HardwareHasAccess(rec, memv)
    img = memv.host_mem.backing
    dev = img.device()
    rng = random.Random(4)
    vas_h = np.array([W.C1_GVA + rng.randrange(64 << 20) if rng.random() < 0.9 else rng.randrange(1 << 32)
                      for _ in range(1 << 20)], dtype=np.uint32)[rank::world]
    vas = torch.from_numpy(vas_h.view(np.int32)).cuda()
    tr = memv.translator(space, use_cache=False)
    tplan = dp.TranslatePlan([tr.device_space], [(0, len(vas_h), 0)], image=img)
    out = (torch.empty(len(vas_h), dtype=torch.int64, device="cuda"),
           torch.empty(len(vas_h), dtype=torch.int32, device="cuda"),
           torch.zeros(len(vas_h), dtype=torch.int64, device="cuda"))
    n_ops, op_len = 4096, 16 << 10
    ops_i = np.arange(n_ops, dtype=np.uint64)[rank::world]
    gv = np.uint64(W.C1_GVA) + ops_i * np.uint64(op_len) + np.uint64(0x40)
    ln = np.full(len(ops_i), op_len - 0x80, dtype=np.uint64)
    offs = np.arange(len(ops_i), dtype=np.uint64) * np.uint64(op_len)
    rows = np.stack([gv, ln, offs, np.zeros(len(ops_i), np.uint64)], 1)
    resolver = acc._resolver
    cplan = dp.CopyPlan([resolver.device_space], rows, shims=[resolver.device_shim])
    src = torch.randint(0, 256, (len(ops_i) * op_len,), dtype=torch.uint8, device="cuda")
    # the shadow leaf nodes, to put the trapping words back between steps
    sroot = space.shadow_root.root_pfn
    leaf_pages = dp.leaf_index(img).leaf_pages([dp.Space(0, sroot)])
    leaf_pages_d = torch.from_numpy(leaf_pages).cuda()
    saved = torch.empty(len(leaf_pages) * 4096, dtype=torch.uint8, device="cuda")
    lib = N.lib()
    stream = torch.cuda.current_stream()
    s = stream.cuda_stream
    N.check(lib.pv_gather_pages(dev.data_ptr(), img.nbytes, leaf_pages_d.data_ptr(), len(leaf_pages),
                                saved.data_ptr(), s), "gather")
    build_s = time.time() - t0

    def restore():
        N.check(lib.pv_scatter_pages(dev.data_ptr(), img.nbytes, leaf_pages_d.data_ptr(), len(leaf_pages),
                                     saved.data_ptr(), s), "scatter")
        img.note_device_write()

    # beside the timed (value, status, aux) walk: the same lanes in 4-byte words, traps (their node pfns)
    # in exception records -- checked equal after the timed steps
    w_words = torch.empty(len(vas_h), dtype=torch.int32, device="cuda")
    w_exc = dp.ExcList(len(vas_h))

    def phase_translate():
        dp.translate_lanes(img, tplan, vas, out=out)

    def phase_copy():
        cplan.shim_written.zero_()
        dp.copy_launch(img, cplan, N.TO_GUEST, src)

    graphs = None

    def step(ev):
        ev[0].record(stream)
        graphs[0].replay() if graphs else phase_translate()
        ev[1].record(stream)
        graphs[1].replay() if graphs else phase_copy()
        ev[2].record(stream)
        img.note_device_write()

    for _ in range(args.warmup):
        restore()
        step([torch.cuda.Event(enable_timing=True) for _ in range(3)])
    torch.cuda.synchronize()
    launch_mode = "eager"
    if not args.no_graph:
        # the two phases as CUDA graphs (same kernels, same arguments every step; the shim's data-dependent
        # work -- which slots trap, which page claims them -- is decided on the device each replay)
        try:
            restore()
            gs = [torch.cuda.CUDAGraph() for _ in range(2)]
            for g, fn in zip(gs, (phase_translate, phase_copy)):
                with torch.cuda.graph(g):
                    fn()
            img.note_device_write()
            torch.cuda.synchronize()
            graphs = gs
            for _ in range(2):
                restore()
                step([torch.cuda.Event(enable_timing=True) for _ in range(3)])
            torch.cuda.synchronize()
            launch_mode = "cuda_graph"
        except Exception as exc:  # noqa: BLE001 - eager launches are the same kernels
            graphs = None
            launch_mode = f"eager (graph capture failed: {type(exc).__name__}: {str(exc)[:120]})"
            torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1 and _pg():
        import torch.distributed as tdist

        tdist.barrier()
    torch.cuda.synchronize()
    fixed = []
    flush = L2Flush()  # 1 M lanes + 64 MiB of copies fit in L2: flushed between steps, outside the events
    for k in range(args.steps):
        restore()
        flush()
        step(evs[k])
        fixed.append(cplan.shim_written.clone())
    torch.cuda.synchronize()
    clk = clocks.stop()
    tr_ms = sum(e[0].elapsed_time(e[1]) for e in evs)
    cp_ms = sum(e[1].elapsed_time(e[2]) for e in evs)
    tr_ms, cp_ms = shard.max_over_ranks([tr_ms, cp_ms], world, device="cuda")
    K = args.steps
    st = out[1].cpu().numpy().view(np.uint32)
    # the same lanes in 4-byte words + exception records decode to exactly the timed step's lanes
    restore()
    w_exc.reset()
    dp.translate_words(img, tplan, vas, w_words, w_exc)
    torch.cuda.synchronize()
    exc, n_exc, overflow = w_exc.read()
    assert not overflow
    wv, ws, wa = dp.unpack_words(w_words.cpu().numpy(), vas_h, exc)
    words_equal = bool(np.array_equal(ws, st) and np.array_equal(wv, out[0].cpu().numpy().view(np.uint64))
                       and np.array_equal(wa, out[2].cpu().numpy().view(np.uint64)))
    assert words_equal, "C4 lane words differ from the (value, status, aux) form"
    kinds = {hex(k): int(c) for k, c in zip(*np.unique(st & 0xFF0, return_counts=True))}
    res = cplan.results.cpu().numpy().view(np.uint64)
    n_fixed = [int(f.item()) for f in fixed]
    assert min(n_fixed) > 0 and len(set(n_fixed)) == 1, n_fixed
    assert 0x10 in [int(k, 16) for k in kinds] and 0x40 in [int(k, 16) for k in kinds]
    total_lanes = 1 << 20
    peak, peak_kind = peaks()
    walk_ach = 16 * len(vas_h) * K / (tr_ms / 1e3) / 1e9
    copied = int(res[:, 0].sum())
    return {
        "metric": METRIC, "value": total_lanes * K / (tr_ms / 1e3), "unit": "translations/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": (tr_ms + cp_ms) / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 (integer walk) / u8 (payload)", "data": "synthetic",
        "config": {"workload": "C4: C1 tables (16,384 shuffled pages), 20 % of shadow leaves not present, 10 % "
                               "trapping; 1 M translations (10 % uniform over 2^32) + 4096 x 16 KiB copy_to_user "
                               "through the hybrid resolver with the device trap shim",
                   "lane_status_counts": kinds, "parallelism": f"lane/op-sharded x{world}", "l2": flush.note()},
        "copy": {"value": copied * K / (cp_ms / 1e3) / 1e9 * world, "unit": "GB/s (payload copied)",
                 "ms_per_step": cp_ms / K, "slots_fixed_by_shim_per_step": n_fixed[0],
                 "ops_faulted": int(((res[:, 3] & 0xFFFFFFFF) != 0).sum())},
        "translate_ms_per_step": tr_ms / K,
        "roofline": {"bound": "hbm", "kernel": "translate_kernel", "achieved": walk_ach, "peak": peak,
                     "unit": "GB/s", "frac": walk_ach / peak, "peak_source": peak_kind,
                     "note": "16 B/translation (u32 VA in, u64 value + u32 status out); 1 M lanes fit L2, so this "
                             "line is latency-bound, not HBM-bound"},
        "walk_form": "unpacked (u64 value + u32 status); the 4-byte word form (one u32 per lane + an exception "
                     "record per trapping lane) is checked equal beside it",
        "exception_records": n_exc, "words_equal_unpacked": words_equal,
        "launch": launch_mode,
        "gpu_launches": 7 * K, "gpu_launches_note": "translate, plan, shim eval + cooperative resolve, stamp, exec per step (+ leaf-index re-encode)",
        "clocks": clk, "build_s": build_s,
        "cpu_baseline": (translate_cpu_baseline(img.host_for_read(), [tr.device_space.s1_base, tr.device_space.s1_root_pfn,
                                                                       0, N.ONE_STAGE], vas_h.astype(np.uint64),
                                                "shadow walks with 30 % corrupted leaves")
                         if rank == 0 and world == 1 and not args.no_cpu_baseline else None),
    }


def run_e2e(wl, args, world):
    """Same step through the public API (ProcessTranslator.translate_batch,
    HardwareHasAccess.copy_to_user_batch) with pinned host buffers: H2D of
    the VAs and payload, D2H of the translations and per-op results are
    inside the timed region."""
    import torch
    import torch.distributed as tdist

    from paper_1304_3771_b200 import has
    from paper_1304_3771_b200 import workloads as W

    memv = wl.memv
    host_vas = [(torch.from_numpy(v.view(np.int32)).pin_memory(), g, p) for g, p, v in wl.proc_vas]
    if wl.name == "c5":
        translators = {(g, p): memv.translator(wl.world.spaces[g][p], use_cache=False)
                       for g, p, _ in wl.proc_vas}
        recs = {}
        for g, p, ops, offs in wl.proc_ops:
            rec = has.GuestProcessRecord(_FakeGuest(g), wl.world.spaces[g][p], memv)
            rec.hybrid = _Prebuilt(wl.world.hybrid_roots[g][p])
            recs[(g, p)] = has.HardwareHasAccess(rec, memv)
    else:
        translators = {(0, 0): memv.translator(wl.c1_space, use_cache=False)}
        rec = has.GuestProcessRecord(_FakeGuest(0, wl.c1_mode), wl.c1_space, memv)
        # hardware HAS needs the shadow table's hybrid root; TDP guests use software HAS (the paper's setup)
        access = has.HardwareHasAccess if wl.c1_mode == "shadow" else has.SoftwareHasAccess
        recs = {(0, 0): access(rec, memv)}
    payload = [(torch.empty(int(ops[:, 1].sum()), dtype=torch.uint8).pin_memory(), g, p, ops)
               for g, p, ops, offs in wl.proc_ops]
    for t, *_ in payload:
        t.random_(0, 256)

    from paper_1304_3771_b200 import dataplane as dp
    from paper_1304_3771_b200 import memvirt as mv

    io = {}
    # results: one pv_translate_words word per lane (the frame number, or the status of the exception
    # the lane raises; the lanes whose exception value is not their own va also return a record) -- 4
    # bytes back per 4-byte VA in.  At N > 1 the words of every rank land in one host buffer all ranks
    # map (shard.SharedHostBuffer): rank 0 holds every guest's results after the step's barrier.
    shared = None
    pg = world > 1 and _pg()
    if pg:
        from paper_1304_3771_b200 import shard as _sh

        shared = _sh.SharedHostBuffer(wl.total_vas * 4, int(os.environ.get("RANK", "0")), world, tag="pv_e2e")
        res_out = [(shared.view(torch.int32, l0, len(v)), None, None)
                   for l0, (_, _, v) in zip(wl.proc_lane0, wl.proc_vas)]
    else:  # caller-owned pinned result buffers, reused every step
        res_out = [(torch.empty(len(v), dtype=torch.int32, pin_memory=True), None, None) for _, _, v in wl.proc_vas]

    def one_step():
        t0 = time.perf_counter()
        io["res"] = mv.translate_many([(translators[(g, p)], t) for t, g, p in host_vas], words=True, out=res_out)
        if pg:
            tdist.barrier()  # every rank's words are in the shared buffer: rank 0 holds all results
        t1 = time.perf_counter()
        # counted from the tensors moved: VAs in; one lane word out -- see dataplane.translate_host_many
        io["h2d"], io["d2h"] = dp.last_host_io["h2d"], dp.last_host_io["d2h"]
        for t, g, p, ops in payload:
            outs = recs[(g, p)].copy_to_user_batch(ops[:, 0], ops[:, 1], t)
            assert all(isinstance(o, int) for o in outs)
        torch.cuda.synchronize()
        return t1 - t0, time.perf_counter() - t1

    one_step()  # warm (pinned pools, plans)
    if world > 1 and _pg():
        tdist.barrier()
    torch.cuda.synchronize()
    tr_s = cp_s = 0.0
    steps = max(1, args.steps)
    tr_each = []
    for _ in range(steps):
        a, b = one_step()
        tr_s += a
        cp_s += b
        tr_each.append(a)
    from paper_1304_3771_b200 import shard

    tr_s, cp_s = shard.max_over_ranks([tr_s, cp_s], world, device="cuda")
    h2d = io["h2d"] + sum(t.numel() for t, *_ in payload)
    d2h = io["d2h"] + sum(len(ops) * 32 for *_, ops in payload)
    # the lane words delivered to the host decode to the device-resident results of the timed step
    # (which verify_parity checked against the oracle)
    dev_v = wl.out[0].cpu().numpy().view(np.uint64)
    dev_s = wl.out[1].cpu().numpy().view(np.uint32)
    lane, same = 0, True
    for (words, _, exc), (t, _, _), (_, _, v) in zip(io["res"], host_vas, wl.proc_vas):
        uv, us, _ = dp.unpack_words(words.numpy(), t.numpy(), exc)
        same &= bool(np.array_equal(uv, dev_v[lane:lane + len(v)]) and np.array_equal(us, dev_s[lane:lane + len(v)]))
        lane += len(v)
    returned = None
    if pg:
        # the words rank 0 reads in the shared buffer are every rank's own results
        mine = hashlib.sha256()
        for l0, (_, _, v) in zip(wl.proc_lane0, wl.proc_vas):
            mine.update(shared.view(torch.int32, l0, len(v)).numpy().tobytes())
        got = [None] * world
        tdist.all_gather_object(got, (mine.hexdigest(), list(zip(wl.proc_lane0, [len(v) for *_, v in wl.proc_vas]))))
        ok = None
        if int(os.environ.get("RANK", "0")) == 0:
            ok = True
            for digest, spans in got:
                h = hashlib.sha256()
                for l0, n in spans:
                    h.update(shared.view(torch.int32, l0, n).numpy().tobytes())
                ok &= h.hexdigest() == digest
        returned = {"to_rank0": "shared host buffer (/dev/shm, cudaHostRegister'd by every rank): each rank's "
                                "D2H writes its guests' lane words where rank 0 reads them; one barrier per step",
                    "bytes": wl.total_vas * 4, "verified": ok}
        shared.close()
    return {"value": wl.total_vas * steps / tr_s, "unit": "translations/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "copy": {"value": wl.total_copy_bytes * steps / cp_s / 1e9, "unit": "GB/s"},
            "steps": steps,
            "translate_ms_per_step": {"mean": 1e3 * tr_s / steps, "best": 1e3 * min(tr_each),
                                      "median": 1e3 * statistics.median(tr_each),
                                      "note": "host-driven pipeline: value uses the mean (max over ranks); best / median "
                                              "over this rank's steps"},
            "results": "one pv_translate_words word per lane (frame number, or status; "
                                       "exception records for lanes whose value is not their va)",
            "lanes_equal_device_results": same,
            "gather_to_rank0": returned,
            "api": "memvirt.translate_many(words=True) (ProcessTranslator.translate_batch over every process) + "
                   "HardwareHasAccess.copy_to_user_batch"}


class _FakeGuest:
    """GuestProcessRecord reads .id and .mem_mode (backend.py:267-286)."""

    def __init__(self, gid, mode: str = "shadow"):
        self.id = gid
        self.mem_mode = mode


class _Prebuilt:
    """A HybridTopLevel that already holds the world's merged root."""

    def __init__(self, root):
        self.root = root

    def build(self, shadow_root, host_root):
        return self.root


def walker_sol(lanes_per_s: float, form: str = "unpacked"):
    """The walker against the measured speed of light of its access pattern
    (random 4-byte gathers + the lane stream: 12 B/lane unpacked, 8 B/lane
    packed, 4 B/lane as words out; profiles/walker_sol.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "walker_sol.json")) as f:
            sol = json.load(f)
    except Exception:  # noqa: BLE001
        return None
    key = {"words": "lanes_per_s_words", "packed": "lanes_per_s_packed"}.get(form, "lanes_per_s")
    if key not in sol:
        return None
    probe = sol[key]
    return {"achieved": lanes_per_s, "probe": probe, "unit": "lanes/s", "frac": lanes_per_s / probe,
            "form": {"words": "words (4 B out)", "packed": "packed (8 B out)"}.get(form, "unpacked (12 B out)"),
            "source": "profiles/walker_sol.json"}


def load_traffic(workload: str) -> dict:
    path = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


def provenance() -> dict:
    """Which code and which device produced this line."""
    import torch

    out = {"gpu": torch.cuda.get_device_name(0) if torch.cuda.is_available() else None}
    try:
        out["git"] = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                                    text=True, timeout=10).stdout.strip() or None
    except Exception:  # noqa: BLE001 - the GPU box's snapshot has no .git
        out["git"] = None
    return out


def load_json_profile(name: str):
    """A committed ncu summary under profiles/ (None when absent)."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return None


def traffic_for(traffic: dict, kernel: str, alg_bytes: int):
    """DRAM bytes per launch of `kernel` from the committed ncu capture,
    scaled to this run's per-launch algorithmic bytes (the capture is the
    N=1 full-size step; a rank at N>1 launches over a 1/N share)."""
    t = traffic.get(kernel)
    a = traffic.get("alg_bytes", {}).get(kernel)
    if t is None or not a:
        return t
    return int(round(t * alg_bytes / a))


def config_of(wl, world):
    if wl.name == "c5":
        c = wl.cfg
        return {"workload": "C5: 8 shadow guests x 8 GiB, 3 processes each, per guest 16M random-VA "
                            "translations + 1 GiB copy_to_user in 4 MiB ops (hybrid/hardware HAS)",
                "guests": c.guests, "guest_bytes": c.guest_bytes, "vas_per_guest": c.vas_per_guest,
                "copy_bytes_per_guest": c.copy_bytes_per_guest, "op_bytes": c.op_bytes,
                "geometry": "reference 3-level 2/9/9/12", "sharding": f"guest g -> rank g mod {world}",
                "parallelism": f"guest-sharded x{world}, no collective",
                "l2": f"inputs larger than L2 ({c.guests * c.vas_per_guest * 4 >> 20} MiB VAs, "
                      f"{c.guests * c.copy_bytes_per_guest >> 20} MiB payload per step, whole job)",
                "scale": 1 if wl.cfg.guest_bytes == 8 << 30 else "reduced"}
    return {"workload": f"C1: 1 {wl.c1_mode} guest, 16384 shuffled pages, 1M random-VA translations + 64 MiB "
                        "copy_to_user", "mode": wl.c1_mode,
            "geometry": "4-level 9/9/9/9/12 (extension, parity unpinned by the reference)" if wl.c1_mode == "4l"
            else "reference 3-level 2/9/9/12",
            "parallelism": f"lane-split x{world} (one process: the VA range and the copy's destination pages "
                           "split evenly over the ranks, image replicated, no collective)",
            "l2": "inputs smaller than L2: L2 flushed between timed steps (256 MiB write outside each step's "
                  "events)"}


# ---- CPU baseline / reference arm ---------------------------------------------------

def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


_SAMPLE_BUF = [None]


def cpu_sample(memv, proc_vas, proc_ops, n_vas: int, n_bytes: int, threads: int):
    """Time the oracle port (oracle/pvoracle.c, test infrastructure) on a
    bounded sample: the first ``n_vas`` translations and ``n_bytes`` of copy
    ops of this workload.  Returns (translations/s, copy GB/s, sample)."""
    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    # the oracle walks the host mirror: bring every table node current first (tables built in HBM
    # reach the host lazily, image.py); C5's nodes all live in the host-private region, the copies
    # only write data pages
    backing = memv.host_mem.backing
    span = getattr(memv, "HOST_PRIVATE_BYTES", backing.nbytes) if backing.nbytes > (4 << 30) else backing.nbytes
    img = backing.host_for_read(0, span)
    # translations: first processes' VAs (shadow walks)
    done = 0
    t_tr = 0.0
    for sp, vas in proc_vas:
        take = vas[: max(0, n_vas - done)]
        if len(take) == 0:
            break
        t0 = time.perf_counter()
        O.translate(img, sp, take.astype(np.uint64), threads=threads)
        t_tr += time.perf_counter() - t0
        done += len(take)
    copied = 0
    t_cp = 0.0
    for sp, ops in proc_ops:
        room = n_bytes - copied
        if room <= 0:
            break
        k = max(1, min(len(ops), room // max(int(ops[0, 1]), 1)))
        sel = ops[:k]
        rows = np.stack([sel[:, 0], sel[:, 1], np.concatenate([[0], np.cumsum(sel[:-1, 1])]).astype(np.uint64),
                         np.zeros(k, np.uint64)], 1).astype(np.uint64)
        need = int(sel[:, 1].sum())
        if _SAMPLE_BUF[0] is None or _SAMPLE_BUF[0].nbytes < need:  # random payload, made once and reused
            _SAMPLE_BUF[0] = np.random.default_rng(0).integers(0, 256, need, dtype=np.uint8)
        buf = _SAMPLE_BUF[0][:need]
        t0 = time.perf_counter()
        O.copy(img, sp.reshape(1, 4), rows, buf, 0, threads=threads)
        t_cp += time.perf_counter() - t0
        copied += int(sel[:, 1].sum())
    return done / t_tr, copied / t_cp / 1e9, f"{done} translations + {copied} bytes of copy_to_user ops"


def _oracle_inputs(wl):
    from oracle import oracle as O

    proc_vas, proc_ops = [], []
    if wl.name == "c5":
        for g, p, v in wl.proc_vas:
            sp = wl.world.spaces[g][p].shadow_root.root_pfn
            proc_vas.append((O.space(0, sp), v))
        for g, p, ops, offs in wl.proc_ops:
            proc_ops.append((O.space(0, wl.world.hybrid_roots[g][p].root_pfn), ops))
    else:
        d = wl.memv.translator(wl.c1_space, use_cache=False).device_space  # shadow or guest + TDP tables
        sp = O.space(d.s1_base, d.s1_root_pfn, d.s2_root_pfn, d.mode)
        proc_vas.append((sp, wl.proc_vas[0][2]))
        proc_ops.append((sp, wl.proc_ops[0][2]))
    return proc_vas, proc_ops


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _pyref_worker(args):
    """One core of the Python reference (devfsim from baseline/_ref, unmodified):
    a shadow guest with 16,384 pages mapped in shuffled order (the C1 world,
    SURVEY.md 8(d)), then the hot loops timed with perf_counter:
    ProcessTranslator.translate (uncached, memvirt.py:585-601) over random VAs
    and HardwareHasAccess.copy_to_user (hybrid resolver, backend.py:152-162)
    of 4 MiB ops at +0x80 (the C5 op shape)."""
    worker, n_vas, n_ops = args
    import random as _r
    import types as _t

    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    from devfsim import backend as rb
    from devfsim import memvirt as rm

    memv = rm.MemoryVirtualizer(host_bytes=128 << 20)
    guest = memv.add_guest(0, "shadow", 96 << 20)
    space = memv.create_process(guest)
    order = list(range(16384))
    _r.Random(1304).shuffle(order)
    for pg in order:
        memv.map_process_page(space, 0x1000_0000 + pg * 4096)
    rng = _r.Random(3771 + worker)
    vas = [0x1000_0000 + rng.randrange(64 << 20) for _ in range(n_vas)]
    tr = memv.translator(space, use_cache=False)
    t0 = time.perf_counter()
    for va in vas:
        tr.translate(va)
    t_tr = time.perf_counter() - t0
    rec = rb.GuestProcessRecord(_t.SimpleNamespace(id=0, mem_mode="shadow"), space, memv)
    acc = rb.HardwareHasAccess(rec, memv)
    data = bytes(rng.randrange(256) for _ in range(4096)) * 1024
    t0 = time.perf_counter()
    for i in range(n_ops):
        acc.copy_to_user(0x1000_0000 + (i % 15) * (4 << 20) + 0x80, data)
    t_cp = time.perf_counter() - t0
    return n_vas / t_tr, n_ops * len(data) / t_cp / 1e9


def _pyref_c2_worker(args):
    """One core of the reference's C2 path (devfsim from baseline/_ref,
    unmodified): a TDP guest (software HAS, blocking transport), the
    EventDevice, one process with a 256-page arena; IOCTL_SNAPSHOT ops with
    arg_len = randint(64, 4096) at arena + randrange(1 MiB - 4096) issued by a
    guest thread through Frontend.vfs_dispatch (frontend.py:124-170 ->
    hypercall -> Backend.execute_fileop, blob staging backend.py:526-534),
    the dispatch loop timed with perf_counter."""
    worker, n_ops = args
    import random as _r

    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    from devfsim.devices import IOCTL_SNAPSHOT, EventDevice
    from devfsim.hypercall import FileOp, FileOpKind
    from devfsim.workloads import open_device
    from devfsim.world import World

    world = World()
    try:
        guest = world.add_guest(vcpus=1, mem_mode="tdp")
        evt = world.add_device(EventDevice(1, "evt", world.clock))
        world.set_mode(guest, evt, "blocking")
        process = world.new_process(guest)
        world.map_buffer(process, 0x2000_0000, 256)
        frontend = world.frontends[guest.id]
        rng = _r.Random(3771 + worker)
        ops = [(0x2000_0000 + rng.randrange((1 << 20) - 4096), rng.randint(64, 4096)) for _ in range(n_ops)]
        box = {}

        def body(t):
            file = frontend.files["/dev/evt"]
            handle = open_device(frontend, t, file)
            t0 = time.perf_counter()
            for gva, ln in ops:
                frontend.vfs_dispatch(t, file, FileOp(kind=FileOpKind.IOCTL, handle=handle, cmd=IOCTL_SNAPSHOT,
                                                      arg_gva=gva, arg_len=ln))
            box["s"] = time.perf_counter() - t0

        thread = world.new_thread(process)
        thread.start(body)
        thread.join(300.0)
        return n_ops / box["s"]
    finally:
        world.close()


def c2_cpu_baseline(memv, spaces, procs, gvas, lens, cores: int, py_ops: int = 1000) -> dict:
    """C2 on the host cores: the oracle port (oracle/pvoracle.c) stages the
    whole trace's blobs -- every op's 2-stage translations through its
    process's FIFO-10 cache, then the copy, in program order per process (one
    thread per process; processes write disjoint arenas) -- and the
    reference's own Python forwarding path is timed per core beside it."""
    import concurrent.futures as cf

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    img = memv.host_mem.backing.host_for_read().copy()
    sp = np.stack([O.space(s.s1_base, s.s1_root_pfn, s.s2_root_pfn, s.mode) for s in
                   (memv.translator(x, use_cache=False).device_space for x in spaces)])
    # every op's blob is the same function of its byte index (devices.py:162-166), so one 4 KiB snapshot
    # serves as every op's source (buffer offset 0): the same bytes as the device payload, 4 KiB of memory
    buf = ((np.arange(4096, dtype=np.int64) * 7 + 3) & 0xFF).astype(np.uint8)
    rows = np.stack([gvas, lens, np.zeros_like(gvas), procs], 1).astype(np.uint64)

    def one(p):
        sel = rows[procs == p]
        cache = O.new_cache(10).reshape(1, -1)
        return O.copy(img, sp, sel, buf, 0, caches=cache, op_cache=np.zeros(len(sel), np.int32))

    n_procs = len(spaces)
    with cf.ThreadPoolExecutor(n_procs) as ex:
        list(ex.map(one, range(n_procs)))  # warm: page-in of the image copy and the payload
        t0 = time.perf_counter()
        res = list(ex.map(one, range(n_procs)))
        dt = time.perf_counter() - t0
    ok = all(((r[:, 3] & 0xFFFFFFFF) == 0).all() for r in res)
    out = {"value": len(gvas) / dt, "unit": "ioctls/s", "cores": n_procs, "kind": "port",
           "sample": f"the whole trace ({len(gvas)} ops): blob staging only (2-stage translations through the "
                     "FIFO-10 caches + copies), one thread per process", "cpu": cpu_model(), "all_ok": bool(ok)}
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "devfsim")):
        import multiprocessing as mp

        t0 = time.perf_counter()
        try:
            with mp.get_context("spawn").Pool(cores) as pool:
                rates = pool.map(_pyref_c2_worker, [(w, py_ops) for w in range(cores)])
            out["python_reference"] = {
                "kind": "reference (devfsim, unmodified pure Python from baseline/_ref)", "cores": cores,
                "ioctls_per_s_per_core": statistics.median(rates), "ioctls_per_s": sum(rates),
                "sample": f"per core: {py_ops} IOCTL_SNAPSHOT ops through Frontend.vfs_dispatch (blocking, TDP "
                          "guest, software HAS): forwarding + driver + blob staging",
                "wall_s": round(time.perf_counter() - t0, 1)}
        except Exception as exc:  # noqa: BLE001 - an optional leg: reported, never fatal to the line
            out["python_reference"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    return out


def python_reference_baseline(cores: int, n_vas: int = 300_000, n_ops: int = 48) -> dict | None:
    try:
        return _python_reference_baseline(cores, n_vas, n_ops)
    except Exception as exc:  # noqa: BLE001 - an optional leg: reported, never fatal to the line
        return {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}


def _python_reference_baseline(cores: int, n_vas: int = 300_000, n_ops: int = 48) -> dict | None:
    """The reference's own CPU path (pure Python, GIL-bound: one process per
    core, SURVEY.md 8(d) "CPU reference timing"), timed on this box beside
    the C port: per-core rates (median over workers) and the K-core
    aggregate.  None when baseline/_ref is not staged."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "devfsim")):
        return None
    import multiprocessing as mp

    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        rows = pool.map(_pyref_worker, [(w, n_vas, n_ops) for w in range(cores)])
    tps = [r[0] for r in rows]
    gbs = [r[1] for r in rows]
    return {"kind": "reference (devfsim, unmodified pure Python from baseline/_ref)", "cores": cores,
            "cpu": cpu_model(),
            "translations_per_s_per_core": statistics.median(tps), "translations_per_s": sum(tps),
            "copy_gbs_per_core": statistics.median(gbs), "copy_gbs": sum(gbs),
            "sample": f"per core: C1 shadow world (16,384 shuffled pages), {n_vas} uncached translate() calls + "
                      f"{n_ops} x 4 MiB HardwareHasAccess.copy_to_user",
            "wall_s": round(time.perf_counter() - t0, 1)}


def translate_cpu_baseline(img: np.ndarray, space_words, vas: np.ndarray, note: str) -> dict:
    """The oracle port's batch translation (oracle/pvoracle.c, all host
    threads) over the same lanes as the device step, one untimed pass then
    the median of three."""
    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    threads = cpu_threads()
    sp = np.asarray(space_words, dtype=np.uint64)
    v = np.ascontiguousarray(vas, dtype=np.uint64)
    O.translate(img, sp, v, threads=threads)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        O.translate(img, sp, v, threads=threads)
        ts.append(time.perf_counter() - t0)
    return {"value": len(v) / statistics.median(ts), "unit": "translations/s", "cores": threads, "kind": "port",
            "sample": f"the step's {len(v)} translations ({note})", "cpu": cpu_model()}


def cpu_baseline(wl, args):
    threads = cpu_threads()
    proc_vas, proc_ops = _oracle_inputs(wl)
    # one untimed pass first: the sample's destination pages are faulted in
    # once (the reference arm's warm-up steps do the same), so both arms time
    # the same steady state
    cpu_sample(wl.memv, proc_vas, proc_ops, args.cpu_sample_vas, args.cpu_sample_bytes, threads)
    # the median of three passes, as the reference arm takes the median of its steps (this box's host
    # cores are a shared 16-CPU slice: single passes vary by +-15 %)
    runs = [cpu_sample(wl.memv, proc_vas, proc_ops, args.cpu_sample_vas, args.cpu_sample_bytes, threads)
            for _ in range(3)]
    tps = statistics.median(r[0] for r in runs)
    gbs = statistics.median(r[1] for r in runs)
    sample = runs[0][2] + " (median of 3 passes)"
    return {"value": tps, "unit": "translations/s", "cores": threads, "kind": "port", "sample": sample,
            "cpu": cpu_model(), "copy": {"value": gbs, "unit": "GB/s"},
            "note": "oracle/pvoracle.c (C restatement of memvirt.py walk/copy_user_buffer, OpenMP, all host "
                    "threads); the reference's own Python path is timed beside it (python_reference)",
            "python_reference": python_reference_baseline(threads)}


class _HostOnlyWorkload:
    """The reference arm's world: host tables only, no device."""

    def __init__(self, name, scale):
        from paper_1304_3771_b200 import workloads as W

        self.name = name
        if name == "c5":
            cfg = W.C5Config() if scale == 1 else W.C5Config().scaled(scale)
            self.cfg = cfg
            self.world = W.build_c5(cfg)
            self.memv = self.world.memv
            self.proc_vas = [(g, p, v) for g in range(cfg.guests) for p, v in enumerate(W.c5_vas(cfg, g))]
            self.proc_ops = [(g, p, ops, None) for g in range(cfg.guests) for p, ops in enumerate(W.c5_ops(cfg, g))]
            self.total_vas = cfg.guests * cfg.vas_per_guest
        else:
            memv, guest, space = W.build_c1("shadow")
            self.memv, self.c1_space = memv, space
            v = W.c1_vas().astype(np.uint32)
            self.proc_vas = [(0, 0, v)]
            self.proc_ops = [(0, 0, np.array([[W.C1_GVA, 64 << 20]], np.uint64), None)]


def run_reference(args, rank, world):
    if rank != 0:
        return None
    wl = _HostOnlyWorkload(args.workload, args.scale)
    threads = cpu_threads()
    proc_vas, proc_ops = _oracle_inputs(wl)
    # the same bounded sample the repo arm's cpu_baseline times (one step = one sample)
    for _ in range(max(args.warmup, 0)):
        cpu_sample(wl.memv, proc_vas, proc_ops, args.cpu_sample_vas, args.cpu_sample_bytes, threads)
    vals, gbs, secs = [], [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        tps, g, sample = cpu_sample(wl.memv, proc_vas, proc_ops, args.cpu_sample_vas, args.cpu_sample_bytes,
                                    threads)
        secs.append(time.perf_counter() - t0)
        vals.append(tps)
        gbs.append(g)
    v = statistics.median(vals)
    return {
        "metric": METRIC, "value": v, "unit": "translations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.median(secs) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "impl": "reference",
        "config": config_of(wl, world) if args.workload == "c5" else {"workload": "C1"},
        "copy": {"value": statistics.median(gbs), "unit": "GB/s"},
        "cpu_baseline": {"value": v, "unit": "translations/s", "cores": threads, "kind": "port", "cpu": cpu_model(),
                         "sample": sample + " per step",
                         "note": "oracle/pvoracle.c: the reference's path restated in C (OpenMP, all host threads), "
                                 "a stronger baseline than the reference's own Python, which is timed beside it",
                         "python_reference": python_reference_baseline(threads)},
        "e2e": {"value": v, "unit": "translations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus != world and world != 1:
        args.gpus = world
    if world > 1 and os.environ.get("PV_BENCH_EMULATE") != "1":
        import torch
        import torch.distributed as tdist

        if args.impl == "ours" and os.environ.get("PV_BENCH_SHARED_DEVICE") != "1":
            torch.cuda.set_device(local)
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group("gloo")
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        runner = {"c2": run_c2, "c3": run_c3, "c4": run_c4}.get(args.workload, run_ours)
        line = runner(args, rank, world, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    bad = line is not None and isinstance(line.get("parity"), dict) and not line["parity"].get("ok", True)
    if world > 1 and _pg():
        import torch.distributed as tdist

        tdist.destroy_process_group()
    if bad:
        sys.exit(f"parity mismatch against the oracle: {line['parity']}")


if __name__ == "__main__":
    main()
