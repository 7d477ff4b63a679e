"""paper_2504_19519_b200 — B200-native FlashOverlap hot path (arXiv 2504.19519).

Thin Python layer over include/flashoverlap.h.  It only marshals arguments
(torch tensors -> device pointers, numpy arrays -> host pointers); every step
of the overlapped GEMM + collective runs in libflashoverlap.so.  PyTorch is
used for device memory, streams and process groups only.

    plan = Plan(coll="allreduce", m=M, n=N, k=K_loc, tile_n=256, workers=S,
                group_waves=[2, 2], rank=r, world=n)
    ctx  = Context.create(device, rank, world, uid)           # NCCL comm + comm stream
    run(ctx, plan, A, Bt, out)                                # overlapped
    run_sequential(ctx, plan, A, Bt, out)                     # GEMM -> one NCCL call
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import COLL, LAYOUT, POST, FOError, check, load

__all__ = ["Plan", "Context", "LoopbackGroup", "run", "run_host", "run_allgather", "rowexchange_stage", "run_sequential", "gemm_stage", "gemm_stage_timed", "post_stage",
           "unique_id", "tune_search", "tune_predict", "kernel_launch_count", "FOError", "load",
           "device_sm_count"]


def _i32(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _p32(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


@dataclass
class PlanSpec:
    coll: str = "allreduce"
    m: int = 0
    n: int = 0
    k: int = 0
    tile_m: int = 128
    tile_n: int = 256
    workers: int = 148
    tile_order: Optional[Sequence[int]] = None
    swizzle: int = 1
    group_waves: Optional[Sequence[int]] = None
    row_dst: Optional[Sequence[int]] = None
    post: str = "none"
    eps: float = 1e-5
    ar_layout: str = "auto"
    a_mn_major: int = 0   # 1: A given as [k, m] row-major (dY of dW = dY^T X)
    b_mn_major: int = 0   # 1: Bt given as [k, n] row-major (X of dW = dY^T X)
    _keep: list = field(default_factory=list, repr=False)

    def to_c(self) -> _lib.PlanDescC:
        order, gw, rd = _i32(self.tile_order), _i32(self.group_waves), _i32(self.row_dst)
        self._keep = [order, gw, rd]
        d = _lib.PlanDescC()
        d.coll = COLL[self.coll]
        d.ar_layout = LAYOUT[self.ar_layout]
        d.m, d.n, d.k = int(self.m), int(self.n), int(self.k)
        d.tile_m, d.tile_n, d.workers = int(self.tile_m), int(self.tile_n), int(self.workers)
        d.tile_order = _p32(order)
        d.swizzle = int(self.swizzle)
        d.num_groups = 0 if gw is None else int(gw.size)
        d.group_waves = _p32(gw)
        d.row_dst = _p32(rd)
        d.post = POST[self.post]
        d.eps = float(self.eps)
        d.a_mn_major = int(self.a_mn_major)
        d.b_mn_major = int(self.b_mn_major)
        return d


class Plan:
    """Host plan of one rank (fo_plan_create).  `peers` (All-to-All only): the
    PlanSpec of every rank, gathered by the caller (see dist.gather_specs)."""

    def __init__(self, rank: int = 0, world: int = 1, peers: Optional[Sequence[PlanSpec]] = None,
                 options: Optional[dict] = None, **kw):
        lib = load()
        self.spec = PlanSpec(**kw)
        self.rank, self.world = rank, world
        d = self.spec.to_c()
        peer_arr = None
        keep = []
        if peers is not None:
            cs = []
            for s in peers:
                s = s if isinstance(s, PlanSpec) else PlanSpec(**s)
                c = s.to_c()
                keep.append(s)
                cs.append(C.pointer(c))
                keep.append(c)
            peer_arr = (C.POINTER(_lib.PlanDescC) * world)(*cs)
        h = C.c_void_p()
        check(lib.fo_plan_create(C.byref(d), rank, world, peer_arr, C.byref(h)))
        self._h = h
        info = _lib.PlanInfoC()
        check(lib.fo_plan_get_info(h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in info._fields_}
        for name, value in (options or {}).items():   # fo_plan_set_option, e.g. {"tail_split": -1}
            self.set_option(name, value)

    @property
    def handle(self):
        return self._h

    def group(self, j: int):
        pb, pe, eb, ee = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
        check(load().fo_plan_group(self._h, j, C.byref(pb), C.byref(pe), C.byref(eb), C.byref(ee)))
        return pb.value, pe.value, eb.value, ee.value

    def export_order(self) -> np.ndarray:
        o = np.empty(self.info["tiles"], np.int32)
        check(load().fo_plan_export_order(self._h, o.ctypes.data_as(C.POINTER(C.c_int32))))
        return o

    def export_send_map(self) -> np.ndarray:
        m = np.empty(self.spec.m * self.spec.n, np.int64)
        check(load().fo_plan_export_send_map(self._h, m.ctypes.data_as(C.POINTER(C.c_int64))))
        return m

    def export_recv_map(self) -> np.ndarray:
        m = np.empty(self.info["out_rows"] * self.info["out_cols"], np.int64)
        check(load().fo_plan_export_recv_map(self._h, m.ctypes.data_as(C.POINTER(C.c_int64))))
        return m

    def export_a2a_counts(self):
        n = self.info["num_groups"] * self.world
        s, r = np.empty(n, np.int64), np.empty(n, np.int64)
        check(load().fo_plan_export_a2a_counts(self._h, s.ctypes.data_as(C.POINTER(C.c_int64)),
                                               r.ctypes.data_as(C.POINTER(C.c_int64))))
        return s.reshape(-1, self.world), r.reshape(-1, self.world)

    def export_calls(self, schedule: int = 0) -> list:
        """The communication calls fo_run (schedule 0) / fo_run_sequential (1)
        issue, in order (fo_plan_export_calls): dicts with kind, group, peer,
        src_buf, dst_buf, src_off, dst_off, count (elements)."""
        lib = load()
        n = C.c_int32()
        check(lib.fo_plan_export_calls(self._h, int(schedule), None, 0, C.byref(n)))
        arr = (_lib.CommCallC * max(1, n.value))()
        check(lib.fo_plan_export_calls(self._h, int(schedule), arr, n.value, C.byref(n)))
        return [dict(kind=_lib.CALL_KINDS[c.kind], group=c.group, peer=c.peer, src_buf=_lib.BUFS[c.src_buf],
                     dst_buf=_lib.BUFS[c.dst_buf], src_off=c.src_off, dst_off=c.dst_off, count=c.count)
                for c in arr[:n.value]]

    def read_counters(self) -> np.ndarray:
        c = np.empty(self.info["num_groups"], np.uint32)
        check(load().fo_plan_read_counters(self._h, c.ctypes.data_as(C.POINTER(C.c_uint32))))
        return c

    def prepare(self, sequential: bool = True, host: bool = False, ctx: "Optional[Context]" = None):
        """fo_plan_prepare: allocate the plan's device state now (tables,
        buffers — registered with `ctx`'s communicator when it registers; the
        sequential / allgather scratch; fo_run_host staging)."""
        check(load().fo_plan_prepare(ctx._h if ctx is not None else None, self._h,
                                     (1 if sequential else 0) | (2 if host else 0)))

    def gemm_cluster(self) -> int:
        """CTAs per cluster of the plan's GEMM launch on the current device (1, 2, 4)."""
        v = C.c_int32(0)
        check(load().fo_plan_gemm_cluster(self._h, C.byref(v)))
        return int(v.value)

    def multicast_used(self) -> bool:
        return self.gemm_cluster() == 4

    def set_debug(self, tile_ts=None, group_ts=None, group_post: int = -1):
        """Evidence hooks: device int64 tensors for tile / group timestamps; group_post -1/0/1."""
        self._dbg = (tile_ts, group_ts)  # keep alive
        check(load().fo_plan_set_debug(self._h, _ptr(tile_ts), _ptr(group_ts), int(group_post)))

    def set_option(self, name: str, value: int):
        """Run-time knobs: group_post (-1/0/1), wait_kernel (0 stream wait, 1 spin kernel)."""
        check(load().fo_plan_set_option(self._h, _lib.OPTION[name], int(value)))

    def fill_buffers(self, pattern: int, stream=None):
        check(load().fo_plan_fill_buffers(self._h, int(pattern) & 0xFFFF, _stream(stream)))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            load().fo_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(load().fo_get_unique_id(buf))
    return bytes(buf)


class Context:
    """Library-owned NCCL communicator + highest-priority comm stream."""

    def __init__(self, handle, device, rank, world):
        self._h, self.device, self.rank, self.world = handle, device, rank, world

    @classmethod
    def create(cls, device: int, rank: int, world: int, uid: bytes, nccl_max_ctas: int = 0, nccl_min_ctas: int = 0,
               cta_policy: str = "default", nvls_ctas: int = 0, buffers: str = "plain") -> "Context":
        """fo_ctx_create_config: the library's NCCL communicator (CTA caps,
        CTA policy, NVLS CTAs) and the buffer registration mode of its plans
        ("plain" cudaMalloc, "registered" ncclMemAlloc + ncclCommRegister,
        "window" ncclMemAlloc + symmetric window registration)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        cfg = _lib.CtxConfigC(int(nccl_max_ctas), int(nccl_min_ctas), _lib.CTA_POLICY[cta_policy], int(nvls_ctas),
                              _lib.BUFFERS[buffers])
        h = C.c_void_p()
        check(load().fo_ctx_create_config(device, rank, world, buf, C.byref(cfg), C.byref(h)))
        ctx = cls(h, device, rank, world)
        ctx.buffers = buffers
        ctx.nccl_max_ctas = int(nccl_max_ctas)
        return ctx

    def mem_alloc(self, shape, dtype=None):
        """A torch tensor on device memory from fo_mem_alloc (ncclMemAlloc,
        registered per the context's buffer mode); freed with the tensor's
        last reference through fo_mem_free."""
        import torch
        dtype = dtype or torch.bfloat16
        n = 1
        for d in shape:
            n *= int(d)
        nbytes = n * torch.empty(0, dtype=dtype).element_size()
        ptr = C.c_void_p()
        check(load().fo_mem_alloc(self._h, int(nbytes), C.byref(ptr)))
        holder = _DeviceBuf(self, ptr.value, tuple(int(d) for d in shape), dtype)
        t = torch.as_tensor(holder, device=torch.device("cuda", self.device))
        return t.view(dtype) if dtype == torch.bfloat16 else t

    @classmethod
    def from_comm(cls, device: int, nccl_comm: int, rank=None, world=None) -> "Context":
        """Context on an existing ncclComm_t (borrowed, never destroyed here);
        the library takes rank and world from the communicator
        (fo_ctx_create_from_comm); `rank`/`world` only label this object."""
        h = C.c_void_p()
        check(load().fo_ctx_create_from_comm(device, C.c_void_p(int(nccl_comm)), C.byref(h)))
        return cls(h, device, rank, world)

    @classmethod
    def loopback(cls, group: "LoopbackGroup", rank: int) -> "Context":
        """TEST backend: rank `rank` of an in-process loopback group on one GPU
        (fo_ctx_create_loopback)."""
        h = C.c_void_p()
        check(load().fo_ctx_create_loopback(group.handle, int(rank), C.byref(h)))
        return cls(h, group.device, rank, group.world)

    @classmethod
    def emulated(cls, device: int, rank: int, world: int, link_gbps: float = 770.0, latency_us: float = 6.0,
                 ctas: int = 16) -> "Context":
        """EVALUATION backend (fo_ctx_create_emulated): rank `rank` of an
        emulated `world`-rank NVLink group on one GPU; collectives take
        latency_us + bus bytes / link_gbps and move their local HBM traffic;
        their results are not the collective's (timing only)."""
        h = C.c_void_p()
        check(load().fo_ctx_create_emulated(int(device), int(rank), int(world), float(link_gbps), float(latency_us),
                                            int(ctas), C.byref(h)))
        ctx = cls(h, device, rank, world)
        ctx.emulated = dict(link_gbps=float(link_gbps), latency_us=float(latency_us), ctas=int(ctas))
        return ctx

    def time_collective_bw(self, coll: str, nbytes: int, iters: int = 5):
        """(average us, bus GB/s) of one collective of `nbytes` (fo_ctx_time_collective)."""
        out, bw = C.c_double(), C.c_double()
        check(load().fo_ctx_time_collective(self._h, COLL[coll], int(nbytes), int(iters), C.byref(out), C.byref(bw)))
        return out.value, bw.value

    def time_collective(self, coll: str, nbytes: int, iters: int = 5) -> float:
        """Average us of one collective of `nbytes` on this context's communicator (tuning)."""
        out = C.c_double()
        check(load().fo_ctx_time_collective(self._h, COLL[coll], int(nbytes), int(iters), C.byref(out), None))
        return out.value

    def sample_curve_bw(self, coll: str, sizes=None, iters: int = 5):
        """(bytes, algorithm GB/s, bus GB/s) samples of `coll` on this communicator."""
        sizes = sizes or [1 << s for s in range(16, 28)]
        out = []
        for sz in sizes:
            us, bus = self.time_collective_bw(coll, sz, iters)
            out.append((sz, sz / (us * 1e-6) / 1e9, bus))
        return out

    def sample_curve(self, coll: str, sizes=None, iters: int = 5):
        """(bytes, GB/s) samples of `coll` on this communicator (Alg. 1 line 5)."""
        sizes = sizes or [1 << s for s in range(16, 28)]
        return [(sz, sz / (self.time_collective(coll, sz, iters) * 1e-6) / 1e9) for sz in sizes]

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            check(load().fo_ctx_destroy(self._h))
            self._h = C.c_void_p()


class _DeviceBuf:
    """__cuda_array_interface__ view of an fo_mem_alloc buffer; frees it (fo_mem_free) when collected."""

    def __init__(self, ctx, ptr, shape, dtype):
        import torch
        self.ctx, self.ptr = ctx, ptr
        # bf16 has no array-interface type string: exposed as int16, viewed back by mem_alloc
        typestr = {torch.bfloat16: "<i2", torch.float16: "<f2", torch.float32: "<f4", torch.int32: "<i4"}[dtype]
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3}
        self._dtype = dtype

    def __del__(self):
        try:
            if self.ctx._h and self.ctx._h.value:
                load().fo_mem_free(self.ctx._h, C.c_void_p(self.ptr))
        except Exception:
            pass


class LoopbackGroup:
    """TEST backend (fo_loopback_create): `world` in-process ranks on one GPU,
    so the multi-rank data path runs on a single-GPU box.  Not for production."""

    def __init__(self, device: int, world: int):
        self.device, self.world = device, world
        h = C.c_void_p()
        check(load().fo_loopback_create(int(device), int(world), C.byref(h)))
        self.handle = h

    def contexts(self):
        return [Context.loopback(self, r) for r in range(self.world)]

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            check(load().fo_loopback_destroy(self.handle))
            self.handle = C.c_void_p()


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)


def run(ctx: Context, plan: Plan, A, Bt, out, residual=None, gamma=None, stream=None):
    check(load().fo_run(ctx._h, plan.handle, _ptr(A), _ptr(Bt), _ptr(out), _ptr(residual), _ptr(gamma),
                        _stream(stream)))


def plan_sync(ctx: Context, plan: Plan, stream=None, timeout_ms: int = 10000):
    """fo_plan_sync: the debug watchdog — wait for the plan's last run with a
    timeout; on timeout the context is aborted and FOError(FO_ERR_TIMEOUT) raised."""
    check(load().fo_plan_sync(ctx._h, plan.handle, _stream(stream), int(timeout_ms)))


def run_host(ctx: Context, plan: Plan, A, Bt, out, residual=None, gamma=None, stream=None):
    """fo_run_host: A, Bt, out (and residual, gamma) are CPU tensors (pin them for async copies)."""
    check(load().fo_run_host(ctx._h, plan.handle, _ptr(A), _ptr(Bt), _ptr(out), _ptr(residual), _ptr(gamma),
                             _stream(stream)))


def run_combine(ctx: Context, plan: Plan, A, Bt, out, idx, w, residual=None, stream=None):
    """fo_run_combine: the A2A plan's overlapped op with the MoE top-k combine
    as its post pass (idx int32 [tokens, k], w float32 [tokens, k], out [tokens, n])."""
    _check_combine(idx, w, out)
    check(load().fo_run_combine(ctx._h, plan.handle, _ptr(A), _ptr(Bt), _ptr(out), _ptr(idx), _ptr(w),
                                int(idx.shape[1]), int(idx.shape[0]), _ptr(residual), _stream(stream)))


def combine_stage(plan: Plan, recv, out, idx, w, residual=None, stream=None):
    """fo_combine_stage: the MoE combine alone on a receive buffer."""
    _check_combine(idx, w, out)
    check(load().fo_combine_stage(plan.handle, _ptr(recv), _ptr(out), _ptr(idx), _ptr(w), int(idx.shape[1]),
                                  int(idx.shape[0]), _ptr(residual), _stream(stream)))


def _check_combine(idx, w, out):
    import torch

    if idx.dtype != torch.int32 or w.dtype != torch.float32 or idx.shape != w.shape or idx.dim() != 2:
        raise ValueError("idx must be int32 [tokens, k] and w float32 of the same shape")
    if out.shape[0] != idx.shape[0]:
        raise ValueError("out must have one row per token")


def run_allgather(ctx: Context, plan: Plan, local, out, residual=None, gamma=None, row_exchange=True, stream=None):
    """RS follow-on: AllGather of the RS outputs (+ row exchange fused with the elementwise op)."""
    check(load().fo_run_allgather(ctx._h, plan.handle, _ptr(local), _ptr(out), _ptr(residual), _ptr(gamma),
                                  int(bool(row_exchange)), _stream(stream)))


def rowexchange_stage(plan: Plan, gathered, out, residual=None, gamma=None, stream=None):
    check(load().fo_rowexchange_stage(plan.handle, _ptr(gathered), _ptr(out), _ptr(residual), _ptr(gamma),
                                      _stream(stream)))


def run_sequential(ctx: Context, plan: Plan, A, Bt, out, residual=None, gamma=None, stream=None):
    check(load().fo_run_sequential(ctx._h, plan.handle, _ptr(A), _ptr(Bt), _ptr(out), _ptr(residual),
                                   _ptr(gamma), _stream(stream)))


def gemm_stage(plan: Plan, A, Bt, send, stream=None):
    check(load().fo_gemm_stage(plan.handle, _ptr(A), _ptr(Bt), _ptr(send), _stream(stream)))


def gemm_stage_timed(plan: Plan, A, Bt, send, tile_ts, stream=None):
    check(load().fo_gemm_stage_timed(plan.handle, _ptr(A), _ptr(Bt), _ptr(send), _ptr(tile_ts), _stream(stream)))


def post_stage(plan: Plan, recv, out, residual=None, gamma=None, stream=None):
    check(load().fo_post_stage(plan.handle, _ptr(recv), _ptr(out), _ptr(residual), _ptr(gamma), _stream(stream)))


def group_post_stage(plan: Plan, j: int, recv, out, residual=None, stream=None):
    """fo_group_post_stage: wave group j's post-reorder alone (the per-group pass of fo_run)."""
    check(load().fo_group_post_stage(plan.handle, int(j), _ptr(recv), _ptr(out), _ptr(residual), _stream(stream)))


def kernel_launch_count() -> int:
    return int(load().fo_kernel_launch_count())


def device_sm_count(device: int = 0) -> int:
    n = C.c_int32()
    check(load().fo_device_sm_count(device, C.byref(n)))
    return n.value


def _curve(curve):
    b = np.ascontiguousarray([float(x) for x, _ in curve], np.float64)
    g = np.ascontiguousarray([float(y) for _, y in curve], np.float64)
    return b, g


def tune_predict(groups, duration_us, tiles, S, tile_bytes, curve) -> float:
    g = _i32(groups)
    b, bw = _curve(curve)
    out = C.c_double()
    check(load().fo_tune_predict(_p32(g), int(g.size), float(duration_us), int(tiles), int(S), float(tile_bytes),
                                 b.ctypes.data_as(C.POINTER(C.c_double)), bw.ctypes.data_as(C.POINTER(C.c_double)),
                                 int(b.size), C.byref(out)))
    return out.value


def tune_search(duration_us, tiles, S, tile_bytes, curve, s1=2, sp=4, prune=True):
    """Alg. 1.  prune: True/1 pruned enumeration, False/0 full enumeration,
    2/3 exact DP argmin without/with the caps (automatic when T > 20)."""
    T = (tiles + S - 1) // S
    b, bw = _curve(curve)
    groups = np.zeros(max(T, 1), np.int32)
    P = C.c_int32()
    pred = C.c_double()
    check(load().fo_tune_search(float(duration_us), int(tiles), int(S), float(tile_bytes),
                                b.ctypes.data_as(C.POINTER(C.c_double)), bw.ctypes.data_as(C.POINTER(C.c_double)),
                                int(b.size), int(s1), int(sp), int(prune), _p32(groups), C.byref(P),
                                C.byref(pred)))
    return tuple(int(x) for x in groups[:P.value]), pred.value


def _d(a):
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def tune_predict_multi(groups, durations, wave_bytes, curve) -> float:
    """A2A imbalance extension: wave_bytes is [ranks][T]."""
    g = _i32(groups)
    wb = np.asarray(wave_bytes, np.float64)
    dur, pd = _d(durations)
    wbf, pw = _d(wb)
    b, bw = _curve(curve)
    out = C.c_double()
    check(load().fo_tune_predict_multi(_p32(g), int(g.size), int(wb.shape[0]), int(wb.shape[1]), pd, pw,
                                       b.ctypes.data_as(C.POINTER(C.c_double)),
                                       bw.ctypes.data_as(C.POINTER(C.c_double)), int(b.size), C.byref(out)))
    return out.value


def tune_search_multi(durations, wave_bytes, curve, s1=2, sp=4, prune=True):
    wb = np.asarray(wave_bytes, np.float64)
    T = int(wb.shape[1])
    dur, pd = _d(durations)
    wbf, pw = _d(wb)
    b, bw = _curve(curve)
    groups = np.zeros(T, np.int32)
    P = C.c_int32()
    pred = C.c_double()
    check(load().fo_tune_search_multi(int(wb.shape[0]), T, pd, pw, b.ctypes.data_as(C.POINTER(C.c_double)),
                                      bw.ctypes.data_as(C.POINTER(C.c_double)), int(b.size), int(s1), int(sp),
                                      int(prune), _p32(groups), C.byref(P), C.byref(pred)))
    return tuple(int(x) for x in groups[:P.value]), pred.value
