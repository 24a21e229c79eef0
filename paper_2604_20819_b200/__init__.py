"""Python binding of libcqs (include/cqs.h): argument marshalling only.

Every step of the hot path (planning, attention, merge, finalize) runs inside libcqs.so; this module
converts Python / torch arguments to the C ABI and raises `CqsError` on any non-OK status.  There is
no fallback: if libcqs.so is missing the import of the library raises immediately.

Same names as the C ABI: cqs_plan, cqs_plan_info, cqs_plan_task, cqs_plan_serialize,
cqs_memory_model, cqs_forward_workspace_size, cqs_attention_forward, cqs_partial_view,
cqs_shard_rows, cqs_merge, cqs_backward_workspace_size, cqs_attention_backward,
cqs_backward_partial_view, cqs_reduce_sum.  `attention()` and
`attention_backward()` are convenience wrappers (allocate the workspace with torch and call the
above).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CQS_LIB") or os.path.join(_HERE, "libcqs.so")  # CQS_LIB: debug variants

CQS_OK, CQS_E_VERIFY, CQS_E_INFEASIBLE, CQS_E_INVALID, CQS_E_CUDA, CQS_E_NCCL, CQS_E_OOM, \
    CQS_E_UNSUPPORTED = range(8)
CQS_F32, CQS_BF16 = 0, 1
CQS_LOC_DEVICE, CQS_LOC_PINNED_HOST = 0, 1
CQS_SCHED_UNIFORM, CQS_SCHED_HYBRID = 0, 1
CQS_SHARD_LPT, CQS_SHARD_CONTIGUOUS = 0, 1
CQS_ACC_BLOCK_ROWS = 256
CQS_PLAN_SUBSET = 1
CQS_MAX_DEPTH, CQS_MAX_SEGS = 12, 32
STATUS_NAMES = {0: "CQS_OK", 1: "CQS_E_VERIFY", 2: "CQS_E_INFEASIBLE", 3: "CQS_E_INVALID",
                4: "CQS_E_CUDA", 5: "CQS_E_NCCL", 6: "CQS_E_OOM", 7: "CQS_E_UNSUPPORTED"}

#: every symbol include/cqs.h declares (tests/test_abi.py checks the .so exports them all)
ABI_SYMBOLS = ("cqs_plan", "cqs_plan_info", "cqs_plan_task", "cqs_plan_serialize",
               "cqs_plan_destroy", "cqs_memory_model", "cqs_forward_workspace_size",
               "cqs_attention_forward", "cqs_partial_view", "cqs_shard_rows", "cqs_merge",
               "cqs_ipc_handle", "cqs_ipc_open", "cqs_ipc_close", "cqs_last_error",
               "cqs_abi_version", "cqs_backward_workspace_size", "cqs_attention_backward",
               "cqs_backward_partial_view", "cqs_reduce_sum", "cqs_partial_runs",
               "cqs_exchange_merge")


class CqsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), msg))
        self.status = status


class PlanDesc(C.Structure):
    _fields_ = [("N", C.c_int64), ("B", C.c_int32), ("H", C.c_int32), ("D", C.c_int32),
                ("c", C.c_int32), ("l", C.c_int32), ("offsets", C.POINTER(C.c_int32)),
                ("depth", C.c_int32), ("budget_bytes", C.c_uint64), ("in_dtype", C.c_int),
                ("out_dtype", C.c_int), ("qkv_loc", C.c_int), ("out_loc", C.c_int),
                ("world", C.c_int32), ("rank", C.c_int32), ("schedule", C.c_int32),
                ("n_level_sets", C.c_int32), ("level_c", C.POINTER(C.c_int32)),
                ("level_offsets", C.POINTER(C.c_int32)), ("shard", C.c_int32),
                ("flags", C.c_int32), ("exec_order", C.POINTER(C.c_int64)),
                ("n_exec_order", C.c_int64), ("n_parallel", C.c_int32),
                ("reserved1", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("depth", C.c_int32), ("acc_depth", C.c_int32), ("n_stage_buffers", C.c_int32),
                ("max_depth", C.c_int32), ("n_tasks", C.c_int64), ("n_empty", C.c_int64),
                ("max_task_rows", C.c_int64), ("max_staged_rows", C.c_int64),
                ("total_work_pairs", C.c_uint64), ("my_tasks", C.c_int64),
                ("my_work_pairs", C.c_uint64), ("dev_workspace_bytes", C.c_uint64),
                ("host_workspace_bytes", C.c_uint64), ("predicted_peak_bytes", C.c_uint64),
                ("acc_rows", C.c_int64), ("shard_rows", C.c_int64)]


class Task(C.Structure):
    _fields_ = [("nseg", C.c_int32), ("rank", C.c_int32), ("depth", C.c_int32),
                ("reserved", C.c_int32), ("work", C.c_uint64),
                ("quorum", C.c_int32 * CQS_MAX_DEPTH), ("seg_start", C.c_int64 * CQS_MAX_SEGS),
                ("seg_len", C.c_int64 * CQS_MAX_SEGS),
                ("seg_codes", (C.c_uint8 * CQS_MAX_DEPTH) * CQS_MAX_SEGS),
                ("kept", C.c_uint32 * CQS_MAX_SEGS)]


class Stats(C.Structure):
    _fields_ = [("ms_plan", C.c_double), ("ms_h2d", C.c_double), ("ms_attn", C.c_double),
                ("ms_merge", C.c_double), ("ms_exchange", C.c_double), ("ms_total", C.c_double),
                ("bytes_h2d", C.c_uint64), ("bytes_d2h", C.c_uint64),
                ("bytes_exchanged", C.c_uint64), ("predicted_peak_bytes", C.c_uint64),
                ("tasks_run", C.c_int64), ("tasks_skipped", C.c_int64),
                ("kernel_launches", C.c_int64)]


_lib = None


def lib():
    """Load libcqs.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libcqs.so not built (run __graft_entry__.build()): " + LIB_PATH)
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.cqs_plan.argtypes = [C.POINTER(PlanDesc), C.POINTER(P)]
        L.cqs_plan_info.argtypes = [P, C.POINTER(PlanInfo)]
        L.cqs_plan_task.argtypes = [P, C.c_int64, C.POINTER(Task)]
        L.cqs_plan_serialize.argtypes = [P, P, C.POINTER(C.c_size_t)]
        L.cqs_plan_destroy.argtypes = [P]
        L.cqs_plan_destroy.restype = None
        L.cqs_memory_model.argtypes = [C.POINTER(PlanDesc), C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.cqs_forward_workspace_size.argtypes = [P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        L.cqs_attention_forward.argtypes = [P, P, P, P, C.POINTER(C.c_int64), P,
                                            C.POINTER(C.c_int64), P, C.c_float, C.c_uint64, P, P,
                                            P, C.POINTER(Stats)]
        L.cqs_partial_view.argtypes = [P, P, C.POINTER(P), C.POINTER(P)]
        L.cqs_shard_rows.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64)]
        L.cqs_merge.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.POINTER(P), C.POINTER(P), P, P, P, C.c_int,
                                C.POINTER(C.c_int64), C.c_int64, C.c_int64, P, P]
        L.cqs_backward_workspace_size.argtypes = [P, C.POINTER(C.c_size_t)]
        L.cqs_attention_backward.argtypes = [P, P, P, P, P, P, C.POINTER(C.c_int64), P, P, P, P,
                                             C.POINTER(C.c_int64), C.c_float, P, P,
                                             C.POINTER(Stats)]
        L.cqs_backward_partial_view.argtypes = [P, P, C.POINTER(P), C.POINTER(P), C.POINTER(P)]
        L.cqs_reduce_sum.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(P), P, C.c_int, C.POINTER(C.c_int64), C.c_int64, P]
        L.cqs_partial_runs.argtypes = [P, C.c_int32, C.c_int64, C.c_int64, C.POINTER(C.c_int64),
                                       C.c_int64, C.POINTER(C.c_int64)]
        L.cqs_exchange_merge.argtypes = [P, C.POINTER(P), C.POINTER(P), C.POINTER(C.c_int64), P,
                                         C.POINTER(C.c_int64), P, P]
        L.cqs_ipc_handle.argtypes = [P, P, C.POINTER(C.c_uint64)]
        L.cqs_ipc_open.argtypes = [P, C.POINTER(P)]
        L.cqs_ipc_close.argtypes = [P]
        L.cqs_last_error.restype = C.c_char_p
        L.cqs_abi_version.restype = C.c_int32
        for name in ABI_SYMBOLS:
            if name not in ("cqs_plan_destroy", "cqs_last_error", "cqs_abi_version"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(st):
    if st != CQS_OK:
        raise CqsError(st, lib().cqs_last_error().decode())


def _i64x4(t):
    return (C.c_int64 * 4)(*[int(x) for x in t])


def _dtype_code(x):
    if isinstance(x, int):
        return x
    return {"bf16": CQS_BF16, "bfloat16": CQS_BF16, "f32": CQS_F32, "float32": CQS_F32}[str(x).replace("torch.", "")]


def _loc_code(x):
    if isinstance(x, int):
        return x
    return {"device": CQS_LOC_DEVICE, "host": CQS_LOC_PINNED_HOST, "pinned": CQS_LOC_PINNED_HOST}[x]


def make_desc(N, B, H, D, depth=1, budget_bytes=0, in_dtype="bf16", out_dtype=None,
              qkv_loc="device", out_loc=None, world=1, rank=0, c=7, offsets=(0, 1, 3),
              schedule="uniform", levels=None, shard="lpt", exec_order=None, subset=False,
              n_parallel=0):
    """levels: optional [(c_t, offsets_t), ...] interest sets for divide levels 0, 1, ...
    (deeper levels use (c, offsets)).  shard: "lpt" | "contiguous" (world > 1 assignment).
    exec_order: optional permutation of the task indices (this rank's execution order); with
    subset=True a list of distinct task indices: only those run (CQS_PLAN_SUBSET).
    n_parallel: tasks in flight on separate streams / accumulator slots (resident plans)."""
    offs = (C.c_int32 * len(offsets))(*offsets)
    levels = list(levels or [])
    lc = (C.c_int32 * max(len(levels), 1))(*[int(c_t) for c_t, _ in levels])
    flat = [int(x) for _, o in levels for x in o]
    lo = (C.c_int32 * max(len(flat), 1))(*flat)
    d = PlanDesc(N=N, B=B, H=H, D=D, c=c, l=len(offsets), offsets=offs, depth=depth,
                 budget_bytes=int(budget_bytes), in_dtype=_dtype_code(in_dtype),
                 out_dtype=_dtype_code(out_dtype if out_dtype is not None else in_dtype),
                 qkv_loc=_loc_code(qkv_loc),
                 out_loc=_loc_code(out_loc if out_loc is not None else qkv_loc),
                 world=world, rank=rank,
                 schedule={"uniform": CQS_SCHED_UNIFORM, "hybrid": CQS_SCHED_HYBRID}.get(
                     schedule, schedule),
                 n_level_sets=len(levels), level_c=lc, level_offsets=lo,
                 shard={"lpt": CQS_SHARD_LPT, "contiguous": CQS_SHARD_CONTIGUOUS}.get(shard, shard),
                 flags=CQS_PLAN_SUBSET if subset else 0, n_parallel=int(n_parallel), reserved1=0)
    eo = None
    if exec_order is not None:
        eo = (C.c_int64 * max(len(exec_order), 1))(*[int(x) for x in exec_order])
        d.exec_order = C.cast(eo, C.POINTER(C.c_int64))
        d.n_exec_order = len(exec_order)
    d._offs = (offs, lc, lo, eo)  # keep alive
    return d


class Plan:
    """Owns a cqs_plan_t*."""

    def __init__(self, desc: PlanDesc):
        self.desc = desc
        h = C.c_void_p()
        _check(lib().cqs_plan(C.byref(desc), C.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.cqs_plan_destroy(self.handle)
            self.handle = None

    def info(self) -> PlanInfo:
        return cqs_plan_info(self)

    def task(self, i) -> Task:
        return cqs_plan_task(self, i)


def cqs_plan(desc=None, **kw) -> Plan:
    return Plan(desc if desc is not None else make_desc(**kw))


def cqs_plan_info(plan: Plan) -> PlanInfo:
    info = PlanInfo()
    _check(lib().cqs_plan_info(plan.handle, C.byref(info)))
    return info


def cqs_plan_task(plan: Plan, idx: int) -> Task:
    t = Task()
    _check(lib().cqs_plan_task(plan.handle, int(idx), C.byref(t)))
    return t


def cqs_plan_serialize(plan: Plan) -> bytes:
    n = C.c_size_t(0)
    _check(lib().cqs_plan_serialize(plan.handle, None, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(lib().cqs_plan_serialize(plan.handle, buf, C.byref(n)))
    return buf.raw[:n.value]


def cqs_memory_model(desc: PlanDesc, depth, acc_depth=0, n_stage_buffers=0):
    dv, hb = C.c_uint64(), C.c_uint64()
    _check(lib().cqs_memory_model(C.byref(desc), depth, acc_depth, n_stage_buffers,
                                  C.byref(dv), C.byref(hb)))
    return dv.value, hb.value


def cqs_forward_workspace_size(plan: Plan):
    dv, hb = C.c_size_t(), C.c_size_t()
    _check(lib().cqs_forward_workspace_size(plan.handle, C.byref(dv), C.byref(hb)))
    return dv.value, hb.value


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def cqs_attention_forward(plan: Plan, q, k, v, out, lse=None, scale=0.0, budget_bytes=0,
                          dev_ws=None, host_ws=None, stream=None, stats=False):
    """q/k/v/out: torch tensors [B,H,N,D] (stride(D)=1); lse: fp32 [B,H,N] contiguous or None.
    k and v must share q's dtype and strides (the C ABI takes one stride array for all three)."""
    import torch
    for t in (k, v):
        if tuple(t.stride()) != tuple(q.stride()) or t.dtype != q.dtype or t.shape != q.shape:
            raise ValueError("q, k, v must share one shape, dtype and layout")
    want = CQS_BF16 if q.dtype == torch.bfloat16 else (CQS_F32 if q.dtype == torch.float32 else -1)
    if want != plan.desc.in_dtype:
        raise ValueError("q dtype %s does not match the plan's in_dtype" % q.dtype)
    if plan.desc.qkv_loc == CQS_LOC_PINNED_HOST and not (q.is_contiguous() and k.is_contiguous()
                                                         and v.is_contiguous()):
        raise ValueError("streamed (pinned host) q, k, v must be contiguous [B,H,N,D]")
    if lse is not None and (lse.dtype != torch.float32 or not lse.is_contiguous()):
        raise ValueError("lse must be a contiguous float32 [B,H,N] tensor")
    st = Stats() if stats else None
    _check(lib().cqs_attention_forward(
        plan.handle, _ptr(q), _ptr(k), _ptr(v), _i64x4(q.stride()), _ptr(out),
        _i64x4(out.stride()) if out is not None else None, _ptr(lse), float(scale),
        int(budget_bytes), _ptr(dev_ws), _ptr(host_ws), _stream_ptr(stream),
        C.byref(st) if st is not None else None))
    return st


def cqs_backward_workspace_size(plan: Plan) -> int:
    dv = C.c_size_t()
    _check(lib().cqs_backward_workspace_size(plan.handle, C.byref(dv)))
    return dv.value


def cqs_attention_backward(plan: Plan, q, k, v, o, dout, lse, dq, dk, dv, scale=0.0, dev_ws=None,
                           stream=None, stats=False):
    """q/k/v/o/dout: bf16 device tensors [B,H,N,D] sharing one layout (stride(D)=1); lse: fp32
    [B,H,N] contiguous (the forward's); dq/dk/dv: [B,H,N,D] of the plan's out dtype, one layout."""
    import torch
    for t in (q, k, v, o, dout):
        if t.dtype != torch.bfloat16:
            raise ValueError("q, k, v, o, dout must be bfloat16 (the backward kernels read bf16)")
    for t in (k, v, o, dout):
        if tuple(t.stride()) != tuple(q.stride()):
            raise ValueError("q, k, v, o, dout must share one layout")
    if lse.dtype != torch.float32 or not lse.is_contiguous():
        raise ValueError("lse must be a contiguous float32 [B,H,N] tensor")
    for t in (dk, dv):
        if dq is not None and tuple(t.stride()) != tuple(dq.stride()):
            raise ValueError("dq, dk, dv must share one layout")
    st = Stats() if stats else None
    _check(lib().cqs_attention_backward(
        plan.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(dout), _i64x4(q.stride()), _ptr(lse),
        _ptr(dq), _ptr(dk), _ptr(dv), _i64x4(dq.stride()) if dq is not None else None,
        float(scale), _ptr(dev_ws), _stream_ptr(stream), C.byref(st) if st is not None else None))
    return st


def cqs_backward_partial_view(plan: Plan, dev_ws):
    """Device addresses of the fp32 dQ, dK, dV accumulators ([N][B*H][D]) inside dev_ws."""
    a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
    _check(lib().cqs_backward_partial_view(plan.handle, _ptr(dev_ws), C.byref(a), C.byref(b),
                                           C.byref(c)))
    return a.value, b.value, c.value


def cqs_reduce_sum(rows, B, H, D, parts, out, out_row0=0, stream=None):
    """out[:, :, out_row0:out_row0+rows] = sum of the fp32 parts ([rows, B*H, D] device tensors
    or raw device addresses, e.g. peer memory), cast to out's dtype."""
    import torch
    n = len(parts)
    pp = (C.c_void_p * max(n, 1))(*[_addr(t) for t in parts])
    od = CQS_BF16 if out.dtype == torch.bfloat16 else CQS_F32
    _check(lib().cqs_reduce_sum(int(rows), B, H, D, n, pp, _ptr(out), od, _i64x4(out.stride()),
                                int(out_row0), _stream_ptr(stream)))


def cqs_partial_view(plan: Plan, dev_ws):
    o, l_ = C.c_void_p(), C.c_void_p()
    _check(lib().cqs_partial_view(plan.handle, _ptr(dev_ws), C.byref(o), C.byref(l_)))
    return o.value, l_.value


def cqs_partial_runs(plan: Plan, src_rank, row0, rows):
    """[(global_start, len, local_row)] of the rows of [row0, row0+rows) that rank src_rank's
    accumulator holds (world > 1: held blocks of CQS_ACC_BLOCK_ROWS rows; world 1: identity)."""
    n = C.c_int64()
    _check(lib().cqs_partial_runs(plan.handle, int(src_rank), int(row0), int(rows), None, 0,
                                  C.byref(n)))
    buf = (C.c_int64 * max(3 * n.value, 1))()
    _check(lib().cqs_partial_runs(plan.handle, int(src_rank), int(row0), int(rows), buf, n.value,
                                  C.byref(n)))
    return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n.value)]


def cqs_exchange_merge(plan: Plan, part_o, part_lse, part_row0, out, lse_out=None, stream=None):
    """The world > 1 exchange merge of this plan's rank: part_o / part_lse = one device address
    (int) or fp32 tensor per rank, part_row0 = the local accumulator row each pointer's row 0 is;
    out: device [B,H,shard_rows,D] (the plan's out dtype), lse_out: device fp32 [B,H,shard_rows]."""
    n = len(part_o)
    po = (C.c_void_p * n)(*[_addr(t) for t in part_o])
    pl = (C.c_void_p * n)(*[_addr(t) for t in part_lse])
    pr = (C.c_int64 * n)(*[int(x) for x in part_row0])
    _check(lib().cqs_exchange_merge(plan.handle, po, pl, pr, _ptr(out), _i64x4(out.stride()),
                                    _ptr(lse_out), _stream_ptr(stream)))


def cqs_shard_rows(N, world, rank):
    a, n = C.c_int64(), C.c_int64()
    _check(lib().cqs_shard_rows(N, world, rank, C.byref(a), C.byref(n)))
    return a.value, n.value


def _addr(x):
    return x if isinstance(x, int) else x.data_ptr()


def cqs_merge(rows, B, H, D, part_o, part_lse, acc_o=None, acc_lse=None, out=None,
              out_row0=0, n_total=None, lse_out=None, stream=None):
    """part_o / part_lse: fp32 device tensors ([rows, B*H, D] / [rows, B*H]) or raw device
    addresses (e.g. peer memory mapped with cqs_ipc_open)."""
    n = len(part_o)
    po = (C.c_void_p * max(n, 1))(*[_addr(t) for t in part_o])
    pl = (C.c_void_p * max(n, 1))(*[_addr(t) for t in part_lse])
    import torch
    od = CQS_BF16 if (out is not None and out.dtype == torch.bfloat16) else CQS_F32
    _check(lib().cqs_merge(int(rows), B, H, D, n, po, pl, _ptr(acc_o), _ptr(acc_lse), _ptr(out), od,
                           _i64x4(out.stride()) if out is not None else None, int(out_row0),
                           int(n_total if n_total is not None else rows), _ptr(lse_out),
                           _stream_ptr(stream)))


def cqs_ipc_handle(dev_ptr: int):
    """(64-byte handle, byte offset) of the device allocation containing dev_ptr."""
    h = C.create_string_buffer(64)
    off = C.c_uint64()
    _check(lib().cqs_ipc_handle(C.c_void_p(dev_ptr), h, C.byref(off)))
    return h.raw, off.value


def cqs_ipc_open(handle: bytes) -> int:
    base = C.c_void_p()
    _check(lib().cqs_ipc_open(C.create_string_buffer(handle, 64), C.byref(base)))
    return base.value


def cqs_ipc_close(base: int):
    _check(lib().cqs_ipc_close(C.c_void_p(base)))


def attention(q, k, v, depth=1, budget_bytes=0, out_dtype=None, scale=0.0, want_lse=True,
              offsets=(0, 1, 3), stats=False):
    """softmax(alpha Q K^T) V for device tensors q, k, v [B,H,N,D] through CQS Divide at `depth`
    (-1: from budget_bytes).  Returns (out, lse[, stats])."""
    import torch
    B, H, N, D = q.shape
    ind = CQS_BF16 if q.dtype == torch.bfloat16 else CQS_F32
    odt = out_dtype or q.dtype
    p = cqs_plan(N=N, B=B, H=H, D=D, depth=depth, budget_bytes=budget_bytes, in_dtype=ind,
                 out_dtype=CQS_BF16 if odt == torch.bfloat16 else CQS_F32, offsets=offsets,
                 c=len(offsets) * (len(offsets) - 1) + 1)
    dev, _ = cqs_forward_workspace_size(p)
    ws = torch.empty(max(dev, 256), dtype=torch.uint8, device=q.device)
    out = torch.empty((B, H, N, D), dtype=odt, device=q.device)
    lse = torch.empty((B, H, N), dtype=torch.float32, device=q.device) if want_lse else None
    st = cqs_attention_forward(p, q, k, v, out, lse, scale, budget_bytes, ws, None, stats=stats)
    return (out, lse, st) if stats else (out, lse)


def attention_backward(q, k, v, o, dout, lse, depth=1, scale=0.0, grad_dtype=None,
                       offsets=(0, 1, 3), stats=False):
    """Gradients (dq, dk, dv) of sum(dout * o) for o = attention(q, k, v) (bf16 device tensors
    [B,H,N,D]; lse the forward's fp32 [B,H,N]) through Algorithm 2 at CQS depth `depth`."""
    import torch
    B, H, N, D = q.shape
    gdt = grad_dtype or q.dtype
    p = cqs_plan(N=N, B=B, H=H, D=D, depth=depth, in_dtype=CQS_BF16,
                 out_dtype=CQS_BF16 if gdt == torch.bfloat16 else CQS_F32, offsets=offsets,
                 c=len(offsets) * (len(offsets) - 1) + 1)
    ws = torch.empty(max(cqs_backward_workspace_size(p), 256), dtype=torch.uint8, device=q.device)
    dq, dk, dv = (torch.empty((B, H, N, D), dtype=gdt, device=q.device) for _ in range(3))
    st = cqs_attention_backward(p, q, k, v, o, dout, lse, dq, dk, dv, scale, ws, stats=stats)
    return (dq, dk, dv, st) if stats else (dq, dk, dv)


def attention_streamed(q, k, v, budget_bytes=0, out_dtype=None, scale=0.0, reserve_bytes=256 << 20,
                       max_retries=6, offsets=(0, 1, 3), stats=False):
    """Streamed forward for q, k, v [B,H,N,D] in PINNED HOST memory; O / lse returned in pinned host
    memory.  OOM guardrail on top of the static plan: the budget defaults to the
    device's free memory minus `reserve_bytes`, and the planner picks the smallest depth, then
    fewer staging buffers (the paper's n_cap - 1), that fits.  If allocating the workspace still
    fails (the budget overstated what the device can give), the budget is re-calibrated from the
    free memory and the plan is rebuilt at least one level deeper (itr + 1), repeatedly.
    Returns (out, lse, info[, stats])."""
    import torch
    B, H, N, D = q.shape
    ind = CQS_BF16 if q.dtype == torch.bfloat16 else CQS_F32
    odt = out_dtype or q.dtype

    def free_budget():
        return max(int(torch.cuda.mem_get_info()[0]) - int(reserve_bytes), 1)

    budget = int(budget_bytes) if budget_bytes else free_budget()
    depth = -1
    for attempt in range(max_retries + 1):
        try:
            p = cqs_plan(N=N, B=B, H=H, D=D, depth=depth, budget_bytes=budget, in_dtype=ind,
                         out_dtype=CQS_BF16 if odt == torch.bfloat16 else CQS_F32,
                         offsets=offsets, c=len(offsets) * (len(offsets) - 1) + 1,
                         qkv_loc="host", out_loc="host")
        except CqsError as e:
            if e.status == CQS_E_INFEASIBLE and depth >= 0 and attempt < max_retries:
                depth += 1                        # explicit depth still too big: one more level
                continue
            raise
        info = p.info()
        dev, host = cqs_forward_workspace_size(p)
        try:
            ws = torch.empty(max(dev, 256), dtype=torch.uint8, device="cuda")
        except torch.cuda.OutOfMemoryError:
            if attempt == max_retries:
                raise
            torch.cuda.empty_cache()
            budget = min(budget, free_budget())   # calibration from what is really free
            depth = info.depth + 1                # guardrail: itr + 1
            continue
        hws = torch.empty(max(host, 256), dtype=torch.uint8).pin_memory() if host else None
        out = torch.empty((B, H, N, D), dtype=odt).pin_memory()
        lse = torch.empty((B, H, N), dtype=torch.float32).pin_memory()
        try:
            st = cqs_attention_forward(p, q, k, v, out, lse, scale, 0, ws, hws, stats=stats)
            torch.cuda.synchronize()
        except CqsError as e:    # a launch ran out of memory (runtime / module memory)
            if e.status != CQS_E_CUDA or "out of memory" not in str(e) or attempt == max_retries:
                raise
            del ws, hws
            torch.cuda.empty_cache()
            budget = min(budget, free_budget())
            depth = info.depth + 1
            continue
        info_d = {"depth": info.depth, "acc_depth": info.acc_depth,
                  "stage_buffers": info.n_stage_buffers, "attempts": attempt + 1,
                  "budget_bytes": int(budget), "workspace_bytes": int(dev)}
        return (out, lse, info_d, st) if stats else (out, lse, info_d)
    raise CqsError(CQS_E_INFEASIBLE, "guardrail: no plan fits after %d retries" % max_retries)


def attention_backward_streamed(q, k, v, o, dout, lse, depth=1, budget_bytes=0, grad_dtype=None,
                                offsets=(0, 1, 3), max_depth_retries=4, stats=False):
    """Backward for q, k, v, o, dout ([B,H,N,D] bf16) and lse ([B,H,N] fp32) in PINNED HOST
    memory; gradients returned in pinned host memory.  If the backward workspace (fp32 gradients
    of all rows + staging) does not fit `budget_bytes` at `depth`, the next depth is tried.
    Returns (dq, dk, dv, info[, stats])."""
    import torch
    B, H, N, D = q.shape
    gdt = grad_dtype or q.dtype
    for attempt in range(max_depth_retries + 1):
        p = cqs_plan(N=N, B=B, H=H, D=D, depth=depth, budget_bytes=budget_bytes,
                     in_dtype=CQS_BF16, out_dtype=CQS_BF16 if gdt == torch.bfloat16 else CQS_F32,
                     offsets=offsets, c=len(offsets) * (len(offsets) - 1) + 1, qkv_loc="host",
                     out_loc="host")
        try:
            need = cqs_backward_workspace_size(p)
            break
        except CqsError as e:
            if e.status != CQS_E_INFEASIBLE or attempt == max_depth_retries:
                raise
            depth = p.info().depth + 1
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device="cuda")
    dq, dk, dv = (torch.empty((B, H, N, D), dtype=gdt).pin_memory() for _ in range(3))
    st = cqs_attention_backward(p, q, k, v, o, dout, lse, dq, dk, dv, 0.0, ws, stats=stats)
    torch.cuda.synchronize()
    info = {"depth": p.info().depth, "workspace_bytes": int(need)}
    return (dq, dk, dv, info, st) if stats else (dq, dk, dv, info)
