"""Thin ctypes binding over libmoe.so (include/moe.h), argument marshalling only.

Every step of the layer runs in the CUDA library; this module passes torch
device pointers and the caller's stream. There is no CPU fallback: if the
library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# MOE_LIB_PATH: development A/B of two builds of this library (tools/ab_lib.sh)
LIB_PATH = os.environ.get("MOE_LIB_PATH") or os.path.join(_PKG, "libmoe.so")

MOE_F_STATS = 1
MOE_F_FORCED_ROUTING = 2
MOE_F_TIMING = 4
MOE_F_NCCL_EXCHANGE = 8
MOE_F_CHECKPOINT = 16
MOE_F_CAC = 32
MOE_F_RANDOM_PRIORITY = 64
MOE_F_AUX_LOSS = 128
MOE_F_NVLS = 256
KERNEL_CLASSES = ("route", "dispatch", "gemm", "combine", "combine_bwd", "gate_bwd", "comm", "xfer")
COLL_NAMES = ("a2a", "allgather", "reducescatter", "allreduce")


class MoEError(RuntimeError):
    def __init__(self, status: int, name: str, detail: str):
        super().__init__(f"{name}: {detail}")
        self.status = status
        self.name = name
        self.detail = detail


class _Config(ctypes.Structure):
    _fields_ = [("tokens", ctypes.c_int64), ("hidden", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("experts", ctypes.c_int32), ("capacity_factor", ctypes.c_float),
                ("g_tensor", ctypes.c_int32), ("g_expert", ctypes.c_int32), ("dtd", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("aux_loss_coef", ctypes.c_float), ("top_k", ctypes.c_int32),
                ("ring_depth", ctypes.c_int32), ("peer_timeout_ms", ctypes.c_int32)]


class _Layout(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("d", ctypes.c_int32),
                ("ep", ctypes.c_int32), ("t", ctypes.c_int32), ("experts_local", ctypes.c_int32),
                ("ffn_local", ctypes.c_int32), ("capacity", ctypes.c_int64),
                ("slot_slice", ctypes.c_int64), ("rows_per_expert", ctypes.c_int64),
                ("token_groups", ctypes.c_int32)]


class _Collective(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pass_", ctypes.c_int32), ("step", ctypes.c_int32),
                ("group_size", ctypes.c_int32), ("buffer_bytes", ctypes.c_int64),
                ("wire_bytes", ctypes.c_int64)]


class _Stats(ctypes.Structure):
    _fields_ = [("calls", ctypes.c_int64 * 4), ("wire_bytes", ctypes.c_int64 * 4),
                ("forward_calls", ctypes.c_int64), ("backward_calls", ctypes.c_int64),
                ("dropped_tokens", ctypes.c_int64), ("tie_tokens", ctypes.c_int64),
                ("nccl_async_error", ctypes.c_int32),
                ("kernel_launches", ctypes.c_int64 * 8), ("kernel_ms", ctypes.c_double * 8),
                ("replay_calls", ctypes.c_int64)]


class _AdamW(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double), ("step", ctypes.c_int64)]


EXPORTS = ("moe_plan_layout", "moe_plan_bytes", "moe_plan_collectives", "moe_get_unique_id",
           "moe_create", "moe_forward", "moe_backward", "moe_forward_replay", "moe_routing", "moe_stats_get",
           "moe_stats_reset", "moe_set_timing", "moe_destroy", "moe_status_string", "moe_last_error_detail",
           "moe_gemm_bf16", "moe_adamw_plan", "moe_adamw_step", "moe_aux_loss", "moe_set_priority_seed",
           "moe_comm_plan_bytes", "moe_comm_create", "moe_comm_destroy", "moe_create_on_comm",
           "moe_emu_group_create", "moe_emu_group_destroy", "moe_comm_create_emulated")
MOE_ERR_STATE = 4
MOE_ERR_TIMEOUT = 8

_lib = None


def lib() -> ctypes.CDLL:
    """Loads libmoe.so (raises if it is missing — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2305_13525_b200.build` "
                           "(the MoE layer has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    cfgp = ctypes.POINTER(_Config)
    L.moe_plan_layout.argtypes = [cfgp, I, I, ctypes.POINTER(_Layout)]
    L.moe_plan_bytes.argtypes = [cfgp, I, I, ctypes.POINTER(SZ), ctypes.POINTER(SZ)]
    L.moe_plan_collectives.argtypes = [cfgp, I, I, ctypes.POINTER(_Collective), I, ctypes.POINTER(I)]
    L.moe_get_unique_id.argtypes = [ctypes.c_char_p]
    L.moe_create.argtypes = [cfgp, ctypes.c_char_p, I, I, P, SZ, ctypes.POINTER(P)]
    L.moe_forward.argtypes = [P, P, P, P, P, P, P, P, P]
    L.moe_backward.argtypes = [P, P, P, P, P, P, P, P, P, P, P, P]
    L.moe_forward_replay.argtypes = [P, P, P, P, P, P, P]
    L.moe_routing.argtypes = [P, P, P, P, P, P, P, P]
    L.moe_stats_get.argtypes = [P, ctypes.POINTER(_Stats)]
    L.moe_stats_reset.argtypes = [P]
    L.moe_set_timing.argtypes = [P, I]
    L.moe_destroy.argtypes = [P]
    L.moe_status_string.argtypes = [I]
    L.moe_status_string.restype = ctypes.c_char_p
    L.moe_last_error_detail.restype = ctypes.c_char_p
    L.moe_gemm_bf16.argtypes = [I, I, I, I, P, I, P, I, P, I, P, I, P]
    I64 = ctypes.c_int64
    L.moe_aux_loss.argtypes = [P, P, P, P]
    L.moe_set_priority_seed.argtypes = [P, ctypes.c_uint64]
    L.moe_adamw_plan.argtypes = [I64, I64, ctypes.POINTER(I64), ctypes.POINTER(SZ)]
    L.moe_adamw_step.argtypes = [P, P, P, P, P, I64, ctypes.POINTER(_AdamW), I64, P, P]
    L.moe_comm_plan_bytes.argtypes = [cfgp, I, I, I, ctypes.POINTER(SZ)]
    L.moe_comm_create.argtypes = [cfgp, I, ctypes.c_char_p, I, I, ctypes.POINTER(P)]
    L.moe_comm_destroy.argtypes = [P]
    L.moe_create_on_comm.argtypes = [cfgp, P, P, SZ, ctypes.POINTER(P)]
    L.moe_emu_group_create.argtypes = [I, ctypes.POINTER(P)]
    L.moe_emu_group_destroy.argtypes = [P]
    L.moe_comm_create_emulated.argtypes = [cfgp, I, P, I, ctypes.POINTER(P)]
    for name in EXPORTS:
        if name not in ("moe_status_string", "moe_last_error_detail"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        L = lib()
        raise MoEError(status, L.moe_status_string(status).decode(), L.moe_last_error_detail().decode())


@dataclass(frozen=True)
class MoEConfig:
    tokens: int
    hidden: int
    ffn: int
    experts: int
    capacity_factor: float = 1.0
    g_tensor: int = 1
    g_expert: int = 1
    dtd: bool = True
    flags: int = MOE_F_STATS
    aux_loss_coef: float = 0.0
    top_k: int = 1
    ring_depth: int = 0          # 0 = 2 forwards in flight per communicator
    peer_timeout_ms: int = 0     # 0 = 60 s deadline per peer barrier / signal wait

    def c(self) -> _Config:
        return _Config(self.tokens, self.hidden, self.ffn, self.experts, self.capacity_factor,
                       self.g_tensor, self.g_expert, int(self.dtd), self.flags, self.aux_loss_coef,
                       self.top_k, self.ring_depth, self.peer_timeout_ms)

    def replace(self, **kw) -> "MoEConfig":
        import dataclasses
        return dataclasses.replace(self, **kw)

    @staticmethod
    def from_shape(shape, dtd: bool = True, forced: bool = False, tokens: int | None = None):
        flags = MOE_F_STATS | (MOE_F_FORCED_ROUTING if forced else 0)
        return MoEConfig(shape.tokens if tokens is None else tokens, shape.hidden, shape.ffn,
                         shape.experts, shape.cf, shape.g_tensor, shape.g_expert, dtd, flags)


def moe_plan_layout(cfg: MoEConfig, world: int = 1, rank: int = 0) -> dict:
    out = _Layout()
    _check(lib().moe_plan_layout(ctypes.byref(cfg.c()), world, rank, ctypes.byref(out)))
    return {k: getattr(out, k) for k, _ in _Layout._fields_}


def moe_plan_bytes(cfg: MoEConfig, world: int = 1, rank: int = 0) -> tuple[int, int]:
    s, c = ctypes.c_size_t(), ctypes.c_size_t()
    _check(lib().moe_plan_bytes(ctypes.byref(cfg.c()), world, rank, ctypes.byref(s), ctypes.byref(c)))
    return s.value, c.value


def moe_plan_collectives(cfg: MoEConfig, world: int = 1, rank: int = 0) -> list[dict]:
    n = ctypes.c_int()
    L = lib()
    _check(L.moe_plan_collectives(ctypes.byref(cfg.c()), world, rank, None, 0, ctypes.byref(n)))
    arr = (_Collective * max(n.value, 1))()
    _check(L.moe_plan_collectives(ctypes.byref(cfg.c()), world, rank, arr, n.value, ctypes.byref(n)))
    return [{"kind": COLL_NAMES[a.kind], "pass": ("forward", "backward", "replay")[a.pass_], "step": a.step,
             "group_size": a.group_size, "buffer_bytes": a.buffer_bytes, "wire_bytes": a.wire_bytes}
            for a in arr[:n.value]]


def _cfg_array(cfgs):
    cfgs = list(cfgs)
    arr = (_Config * len(cfgs))(*[c.c() for c in cfgs])
    return arr, len(cfgs)


def moe_comm_plan_bytes(cfgs, world: int, rank: int = 0) -> int:
    """Device bytes of the peer windows a communicator for these layers allocates."""
    arr, n = _cfg_array(cfgs)
    out = ctypes.c_size_t()
    _check(lib().moe_comm_plan_bytes(arr, n, world, rank, ctypes.byref(out)))
    return out.value


class MoEComm:
    """A communicator shared by the MoE layers of one process (moe_comm_create), or one
    rank of an emulated group (EmuGroup.comm). Layers attach with MoELayer(..., comm=)."""

    def __init__(self, cfgs, world: int, rank: int, emu: "EmuGroup | None" = None):
        self.world, self.rank = world, rank
        self.cfgs = list(cfgs)
        arr, n = _cfg_array(self.cfgs)
        h = ctypes.c_void_p()
        if emu is not None:
            _check(lib().moe_comm_create_emulated(arr, n, emu.h, rank, ctypes.byref(h)))
        else:
            import torch.distributed as dist
            obj = [moe_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            _check(lib().moe_comm_create(arr, n, obj[0], world, rank, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            _check(lib().moe_comm_destroy(self.h))
            self.h = ctypes.c_void_p()


class EmuGroup:
    """`world` ranks emulated in this process on the current device (moe_emu_group):
    every rank runs on its own Python thread and stream (ctypes releases the GIL)."""

    def __init__(self, world: int):
        self.world = world
        h = ctypes.c_void_p()
        _check(lib().moe_emu_group_create(world, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().moe_emu_group_destroy(self.h)
            self.h = ctypes.c_void_p()


def moe_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().moe_get_unique_id(buf))
    return buf.raw


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def moe_gemm_bf16(A, B, D, a_mn: int, b_mn: int, epilogue: int = 0, aux=None, impl: int = 0,
                  stream=None):
    """D[b] = epi(A[b] . B[b]^T) — layouts per include/moe.h (diagnostic entry point)."""
    batch = D.shape[0]
    M, N = D.shape[1], D.shape[2]
    K = A.shape[2] if not a_mn else A.shape[1]
    _check(lib().moe_gemm_bf16(batch, M, N, K, _ptr(A), a_mn, _ptr(B), b_mn, _ptr(D), epilogue,
                               _ptr(aux), impl, _stream(stream)))


MOE_TILE_PARAMS_PAPER = 1_800_000  # include/moe_optim.h


def moe_adamw_plan(n: int, tile_params: int):
    """(n_tiles, temp_bytes) of the tiled optimizer step (include/moe_optim.h)."""
    nt, tb = ctypes.c_int64(), ctypes.c_size_t()
    _check(lib().moe_adamw_plan(n, tile_params, ctypes.byref(nt), ctypes.byref(tb)))
    return nt.value, tb.value


def moe_adamw_step(grad, master, exp_avg, exp_avg_sq, param=None, *, lr: float, beta1: float,
                   beta2: float, eps: float, weight_decay: float, step: int, tile_params: int = 0,
                   temp=None, stream=None):
    """One AdamW step of include/moe_optim.h: grad/param bf16, the rest fp32, same numel;
    tile_params > 0 runs the paper's tiled step with `temp` (fp32, >= plan temp bytes)."""
    n = master.numel()
    h = _AdamW(lr, beta1, beta2, eps, weight_decay, step)
    _check(lib().moe_adamw_step(_ptr(grad), _ptr(master), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(param), n,
                                ctypes.byref(h), tile_params, _ptr(temp), _stream(stream)))


class MoELayer:
    """One rank's MoE layer context (moe_create / moe_forward / moe_backward).

    For world > 1 the NCCL unique id is broadcast with torch.distributed
    (the default process group, any backend) before moe_create.
    """

    def __init__(self, cfg: MoEConfig, world: int = 1, rank: int = 0, device=None,
                 comm: MoEComm | None = None):
        self.cfg = cfg
        if comm is not None:
            world, rank = comm.world, comm.rank
        self.world, self.rank = world, rank
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.layout = moe_plan_layout(cfg, world, rank)
        self.saved_bytes, self.scratch_bytes = moe_plan_bytes(cfg, world, rank)
        self.scratch = torch.empty(max(self.scratch_bytes, 256), dtype=torch.uint8, device=self.device)
        self.comm = comm
        if comm is not None:
            ctx = ctypes.c_void_p()
            _check(lib().moe_create_on_comm(ctypes.byref(cfg.c()), comm.h, _ptr(self.scratch),
                                            self.scratch_bytes, ctypes.byref(ctx)))
            self.ctx = ctx
            return
        uid = bytes(128)
        if world > 1:
            import torch.distributed as dist
            obj = [moe_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        ctx = ctypes.c_void_p()
        _check(lib().moe_create(ctypes.byref(cfg.c()), uid, world, rank, _ptr(self.scratch),
                                self.scratch_bytes, ctypes.byref(ctx)))
        self.ctx = ctx

    def new_saved(self) -> torch.Tensor:
        return torch.empty(self.saved_bytes, dtype=torch.uint8, device=self.device)

    def moe_forward(self, x, wg, w1, w2, y=None, saved=None, forced=None, stream=None):
        y = torch.empty_like(x) if y is None else y
        saved = self.new_saved() if saved is None else saved
        _check(lib().moe_forward(self.ctx, _ptr(x), _ptr(wg), _ptr(w1), _ptr(w2), _ptr(y),
                                 _ptr(saved), _ptr(forced), _stream(stream)))
        return y, saved

    def moe_backward(self, dy, saved, x, wg, w1, w2, out=None, stream=None):
        if out is None:
            out = (torch.empty_like(x), torch.empty_like(wg), torch.empty_like(w1), torch.empty_like(w2))
        dx, dwg, dw1, dw2 = out
        _check(lib().moe_backward(self.ctx, _ptr(dy), _ptr(saved), _ptr(x), _ptr(wg), _ptr(w1),
                                  _ptr(w2), _ptr(dx), _ptr(dwg), _ptr(dw1), _ptr(dw2), _stream(stream)))
        return dx, dwg, dw1, dw2

    def moe_forward_replay(self, saved, x, wg, w1, w2, stream=None):
        _check(lib().moe_forward_replay(self.ctx, _ptr(saved), _ptr(x), _ptr(wg), _ptr(w1), _ptr(w2),
                                        _stream(stream)))

    def moe_routing(self, saved, stream=None) -> dict:
        """expert/slot/prob: [T] (top-1) or [T, 2] (top-2); gap [T]; count [E]."""
        T, E = self.cfg.tokens, self.cfg.experts
        dev = self.device
        shp = (T, 2) if self.cfg.top_k == 2 else (T,)
        out = {"expert": torch.empty(shp, dtype=torch.int32, device=dev),
               "slot": torch.empty(shp, dtype=torch.int32, device=dev),
               "prob": torch.empty(shp, dtype=torch.float32, device=dev),
               "gap": torch.empty(T, dtype=torch.float32, device=dev),
               "count": torch.empty(E, dtype=torch.int32, device=dev)}
        _check(lib().moe_routing(self.ctx, _ptr(saved), _ptr(out["expert"]), _ptr(out["slot"]),
                                 _ptr(out["prob"]), _ptr(out["gap"]), _ptr(out["count"]), _stream(stream)))
        return out

    def moe_aux_loss(self, saved, stream=None) -> torch.Tensor:
        """MOE_F_AUX_LOSS: this forward's l_aux as a 1-element fp32 device tensor."""
        out = torch.empty(1, dtype=torch.float32, device=self.device)
        _check(lib().moe_aux_loss(self.ctx, _ptr(saved), _ptr(out), _stream(stream)))
        return out

    def moe_set_priority_seed(self, seed: int):
        """MOE_F_RANDOM_PRIORITY: key of the priority permutation for later forwards."""
        _check(lib().moe_set_priority_seed(self.ctx, seed & ((1 << 64) - 1)))

    def moe_stats(self) -> dict:
        s = _Stats()
        _check(lib().moe_stats_get(self.ctx, ctypes.byref(s)))
        return {"calls": dict(zip(COLL_NAMES, list(s.calls))),
                "wire_bytes": dict(zip(COLL_NAMES, list(s.wire_bytes))),
                "forward_calls": s.forward_calls, "backward_calls": s.backward_calls,
                "dropped_tokens": s.dropped_tokens, "tie_tokens": s.tie_tokens,
                "nccl_async_error": s.nccl_async_error,
                "kernel_launches": dict(zip(KERNEL_CLASSES, list(s.kernel_launches))),
                "kernel_ms": dict(zip(KERNEL_CLASSES, list(s.kernel_ms))),
                "replay_calls": s.replay_calls}

    def moe_stats_reset(self):
        _check(lib().moe_stats_reset(self.ctx))

    def moe_set_timing(self, on: bool):
        _check(lib().moe_set_timing(self.ctx, 1 if on else 0))

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            lib().moe_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MoEFunction(torch.autograd.Function):
    """autograd wrapper: y = MoE(x; wg, w1, w2) through moe_forward/moe_backward."""

    @staticmethod
    def forward(ctx, layer: MoELayer, x, wg, w1, w2):
        y, saved = layer.moe_forward(x, wg, w1, w2)
        ctx.layer = layer
        ctx.save_for_backward(x, wg, w1, w2, saved)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, wg, w1, w2, saved = ctx.saved_tensors
        dx, dwg, dw1, dw2 = ctx.layer.moe_backward(dy.contiguous(), saved, x, wg, w1, w2)
        return None, dx, dwg, dw1, dw2
