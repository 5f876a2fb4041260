"""ctypes binding of libspa.so (include/spa.h): argument marshalling only.

Every step of the path runs in the library's CUDA kernels / NCCL calls.  There is no
fallback: if libspa.so is missing or fails to load, importing the functions raises.
torch is used for device memory and streams only (tensor.data_ptr(), stream.cuda_stream).
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import List, Optional, Sequence

from . import _build

__all__ = [
    "SpaError", "load", "header_functions", "get_unique_id", "Comm", "Plan", "Shape", "Profile",
    "spa_attention_fwd", "spa_attention_fwd_masked", "spa_attention_fwd_ex", "attention_fp32", "spa_pipesp_attention", "spa_ulysses_attention", "spa_aco_attention",
    "spa_pipesp_attention_local", "spa_ulysses_attention_local", "spa_aco_attention_local",
    "spa_ring_attention", "spa_ring_attention_local", "spa_attention_host",
    "spa_reshard_seq_to_head", "spa_reshard_head_to_seq", "spa_reshard_seq_to_head_local",
    "spa_reshard_head_to_seq_local", "spa_pad_heads", "attention", "BUF_Q", "BUF_K", "BUF_V", "BUF_OUT",
    "BUF_WS", "SPA_OPT_PROFILE", "SPA_OPT_SKIP_COMM", "SPA_OPT_COPROC_BUSY", "SPA_OPT_DIRECT", "SPA_OPT_COMM_SMS",
    "SPA_OPT_RANK_ONLY", "SPA_OPT_LOOPBACK_CE", "SPA_OPT_STAGE_WINDOW",
    "spa_pipesp_qkv_attention", "spa_pipesp_qkv_attention_local", "spa_qkv_projection",
    "spa_pipesp_attention_hostbuf", "spa_pipesp_attention_hostbuf_local",
]

SPA_OPT_PROFILE, SPA_OPT_SKIP_COMM, SPA_OPT_COPROC_BUSY, SPA_OPT_DIRECT, SPA_OPT_COMM_SMS = 1, 2, 3, 4, 5
SPA_OPT_RANK_ONLY, SPA_OPT_LOOPBACK_CE, SPA_OPT_STAGE_WINDOW = 6, 7, 8
BUF_Q, BUF_K, BUF_V, BUF_OUT, BUF_WS = 0, 1, 2, 3, 4
HEADER = os.path.join(os.path.dirname(_build.HERE), "include", "spa.h")


class SpaError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__(f"{where}: {_status_name(status)}: {detail}")


class Shape(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int), ("S", ctypes.c_int), ("H", ctypes.c_int), ("D", ctypes.c_int),
                ("stages", ctypes.c_int), ("n_src", ctypes.c_int), ("pad_heads", ctypes.c_int),
                ("ring", ctypes.c_int), ("ulysses", ctypes.c_int)]


class CommConfig(ctypes.Structure):
    _fields_ = [("min_ctas", ctypes.c_int), ("max_ctas", ctypes.c_int), ("cta_policy", ctypes.c_int)]


class Profile(ctypes.Structure):
    _fields_ = [("n_stages", ctypes.c_int), ("total_ms", ctypes.c_float), ("pack_ms", ctypes.c_float),
                ("unpack_ms", ctypes.c_float), ("attn_ms", ctypes.c_float * 64),
                ("a2a_in_ms", ctypes.c_float * 64), ("a2a_out_ms", ctypes.c_float * 64),
                ("attn_launches", ctypes.c_int), ("copy_launches", ctypes.c_int), ("gemm_launches", ctypes.c_int)]


class CopyDesc(ctypes.Structure):
    _fields_ = [("src_buf", ctypes.c_int), ("dst_buf", ctypes.c_int), ("src_rank", ctypes.c_int),
                ("dst_rank", ctypes.c_int), ("src_off", ctypes.c_longlong), ("dst_off", ctypes.c_longlong),
                ("count", ctypes.c_longlong * 4), ("src_stride", ctypes.c_longlong * 4),
                ("dst_stride", ctypes.c_longlong * 4), ("run_bytes", ctypes.c_longlong)]


class Msg(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int), ("is_recv", ctypes.c_int), ("buf", ctypes.c_int),
                ("off", ctypes.c_longlong), ("bytes", ctypes.c_longlong)]


class AttnDesc(ctypes.Structure):
    _fields_ = [("q_off", ctypes.c_longlong), ("k_off", ctypes.c_longlong), ("v_off", ctypes.c_longlong),
                ("o_off", ctypes.c_longlong), ("B", ctypes.c_int), ("Sq", ctypes.c_int), ("Skv", ctypes.c_int),
                ("n_heads", ctypes.c_int), ("q_tok_stride", ctypes.c_longlong),
                ("q_batch_stride", ctypes.c_longlong), ("kv_tok_stride", ctypes.c_longlong),
                ("kv_batch_stride", ctypes.c_longlong)]


_lib = None
_P = ctypes.c_void_p
_PP = ctypes.POINTER(ctypes.c_void_p)
_LL = ctypes.c_longlong


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libspa.so (building it in-tree with nvcc if absent).  Raises if that fails."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SPA_LIB") or _build.LIB   # SPA_LIB: debug builds (lib/libspa_trace.so)
    if not os.path.exists(path):
        if not build_if_missing:
            raise OSError(f"libspa.so not built: {path}")
        _build.build()
    lib = ctypes.CDLL(path)
    i, ip = ctypes.c_int, ctypes.POINTER(ctypes.c_int)
    sig = {
        "spa_version": ([], ctypes.c_char_p),
        "spa_status_string": ([i], ctypes.c_char_p),
        "spa_last_error": ([], ctypes.c_char_p),
        "spa_pad_heads": ([i, i, ip], i),
        "spa_get_unique_id": ([ctypes.c_char_p], i),
        "spa_comm_init": ([_PP, ctypes.c_char_p, i, i, i], i),
        "spa_comm_init_loopback": ([_PP, i, i], i),
        "spa_comm_init_host": ([_PP, i, i], i),
        "spa_comm_init_p2p": ([_PP, i, i, i], i),
        "spa_comm_init_config": ([_PP, ctypes.c_char_p, i, i, i, ctypes.POINTER(CommConfig)], i),
        "spa_comm_wait": ([_P, _P, i], i),
        "spa_plan_ipc_handle": ([_P, _P, ctypes.c_char_p], i),
        "spa_plan_ipc_open": ([_P, _P, ctypes.c_char_p], i),
        "spa_mem_alloc": ([ctypes.c_size_t, _PP], i),
        "spa_mem_free": ([_P], i),
        "spa_plan_window_register": ([_P, _P], i),
        "spa_comm_window_selftest": ([_P, ctypes.c_size_t], i),
        "spa_comm_split": ([_P, i, i, _PP], i),
        "spa_comm_check": ([_P], i),
        "spa_comm_destroy": ([_P], i),
        "spa_comm_info": ([_P, ip, ip, ip], i),
        "spa_plan_create": ([_PP, _P, ctypes.POINTER(Shape)], i),
        "spa_plan_workspace_bytes": ([_P, ctypes.POINTER(ctypes.c_size_t)], i),
        "spa_plan_stage_split": ([_P, ip, ip, ip], i),
        "spa_plan_destroy": ([_P], i),
        "spa_plan_set_option": ([_P, i, i], i),
        "spa_plan_set_kv_len": ([_P, _P], i),
        "spa_plan_last_profile": ([_P, ctypes.POINTER(Profile)], i),
        "spa_ulysses_attention": ([_P, _P, _P, _P, _P, _P, _P], i),
        "spa_pipesp_attention": ([_P, _P, _P, _P, _P, _P, _P], i),
        "spa_aco_attention": ([_P, _P, _P, _P, _P, _P, _P], i),
        "spa_ulysses_attention_local": ([_P, _PP, _PP, _PP, _PP, _P, _P], i),
        "spa_pipesp_attention_local": ([_P, _PP, _PP, _PP, _PP, _P, _P], i),
        "spa_aco_attention_local": ([_P, _PP, _PP, _PP, _PP, _P, _P], i),
        "spa_ring_attention": ([_P, _P, _P, _P, _P, _P, _P], i),
        "spa_attention_host": ([_P, _P, _P, _P, _P, _P, _P], i),
        "spa_plan_host_sp_workspace_bytes": ([_P, ctypes.POINTER(ctypes.c_size_t)], i),
        "spa_pipesp_attention_hostbuf": ([_P, _P, _P, _P, _P, _P, _P], i),
        "spa_pipesp_attention_hostbuf_local": ([_P, _PP, _PP, _PP, _PP, _P, _P], i),
        "spa_plan_host_workspace_bytes": ([_P, ctypes.POINTER(ctypes.c_size_t)], i),
        "spa_ring_attention_local": ([_P, _PP, _PP, _PP, _PP, _P, _P], i),
        "spa_reshard_seq_to_head": ([_P, _P, _P, _P, _P], i),
        "spa_reshard_head_to_seq": ([_P, _P, _P, _P, _P], i),
        "spa_reshard_seq_to_head_local": ([_P, _PP, _PP, _P, _P], i),
        "spa_reshard_head_to_seq_local": ([_P, _PP, _PP, _P, _P], i),
        "spa_attention_fwd": ([_P, _P, _P, _P, i, i, i, i, i, _LL, _LL, _LL, _LL, _LL, _LL, _P], i),
        "spa_attention_fwd_masked": ([_P, _P, _P, _P, i, i, i, i, i, _LL, _LL, _LL, _LL, _LL, _LL, _P, _P], i),
        "spa_attention_fwd_ex": ([_P, _P, _P, _P, i, i, i, i, i, _LL, _LL, _LL, _LL, _LL, _LL, _P, i, _P, _P], i),
        "spa_plan_describe_pack": ([_P, i, ctypes.POINTER(CopyDesc), i, ip], i),
        "spa_plan_describe_unpack": ([_P, i, ctypes.POINTER(CopyDesc), i, ip], i),
        "spa_plan_describe_messages": ([_P, i, i, i, ctypes.POINTER(Msg), i, ip], i),
        "spa_plan_describe_attention": ([_P, i, i, ctypes.POINTER(AttnDesc)], i),
        "spa_plan_describe_ring": ([_P, i, i, ctypes.POINTER(Msg), i, ip], i),
        "spa_plan_qkv_weight_bytes": ([_P, i, ctypes.POINTER(ctypes.c_size_t)], i),
        "spa_plan_qkv_workspace_bytes": ([_P, ctypes.POINTER(ctypes.c_size_t)], i),
        "spa_plan_pack_qkv_weight": ([_P, i, _P, _P, _P, _P], i),
        "spa_pipesp_qkv_attention": ([_P, i, _P, _P, _P, _P, _P], i),
        "spa_pipesp_qkv_attention_local": ([_P, i, _PP, _P, _PP, _P, _P], i),
        "spa_qkv_projection": ([_P, i, i, _P, _P, _P, _P, _P, _P], i),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def header_functions() -> List[str]:
    """Function names declared in include/spa.h."""
    with open(HEADER) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spa_[a-z0-9_]+)\s*\(", text)))


def _status_name(s: int) -> str:
    try:
        return load().spa_status_string(s).decode()
    except Exception:  # pragma: no cover
        return str(s)


def _check(status: int, where: str):
    if status != 0:
        raise SpaError(status, where, load().spa_last_error().decode(errors="replace"))


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _arr(ptrs: Sequence) -> ctypes.Array:
    return (ctypes.c_void_p * len(ptrs))(*[_ptr(p) for p in ptrs])


def spa_pad_heads(H: int, n: int):
    pad = ctypes.c_int(0)
    hp = load().spa_pad_heads(H, n, ctypes.byref(pad))
    return hp, pad.value


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().spa_get_unique_id(buf), "spa_get_unique_id")
    return buf.raw


class Comm:
    """spa_comm wrapper.  Use Comm.nccl(...), Comm.loopback(...) or Comm.host(...)."""

    def __init__(self, handle: int):
        self.h = ctypes.c_void_p(handle)
        n, r, k = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(load().spa_comm_info(self.h, ctypes.byref(n), ctypes.byref(r), ctypes.byref(k)), "spa_comm_info")
        self.nranks, self.rank, self.kind = n.value, r.value, k.value

    @classmethod
    def nccl(cls, uid: bytes, nranks: int, rank: int, device: int, min_ctas: int = 0, max_ctas: int = 0,
             cta_policy: int = 0) -> "Comm":
        h = ctypes.c_void_p()
        if min_ctas or max_ctas or cta_policy:
            cfg = CommConfig(min_ctas, max_ctas, cta_policy)
            _check(load().spa_comm_init_config(ctypes.byref(h), uid, nranks, rank, device, ctypes.byref(cfg)),
                   "spa_comm_init_config")
        else:
            _check(load().spa_comm_init(ctypes.byref(h), uid, nranks, rank, device), "spa_comm_init")
        return cls(h.value)

    def wait(self, stream=None, timeout_ms: int = -1):
        """Block until `stream` completes; a failed peer or the timeout aborts the NCCL communicator (SpaError)."""
        _check(load().spa_comm_wait(self.h, _stream(stream), timeout_ms), "spa_comm_wait")

    @classmethod
    def loopback(cls, nvirtual: int, device: int = 0) -> "Comm":
        h = ctypes.c_void_p()
        _check(load().spa_comm_init_loopback(ctypes.byref(h), nvirtual, device), "spa_comm_init_loopback")
        return cls(h.value)

    @classmethod
    def p2p(cls, nranks: int, rank: int, device: int) -> "Comm":
        """One process per rank, exchange over CUDA IPC peer memory (no NCCL); see Plan.ipc_setup."""
        h = ctypes.c_void_p()
        _check(load().spa_comm_init_p2p(ctypes.byref(h), nranks, rank, device), "spa_comm_init_p2p")
        return cls(h.value)

    @classmethod
    def host(cls, nranks: int, rank: int) -> "Comm":
        h = ctypes.c_void_p()
        _check(load().spa_comm_init_host(ctypes.byref(h), nranks, rank), "spa_comm_init_host")
        return cls(h.value)

    def split(self, color: int, key: int) -> Optional["Comm"]:
        h = ctypes.c_void_p()
        _check(load().spa_comm_split(self.h, color, key, ctypes.byref(h)), "spa_comm_split")
        return Comm(h.value) if h.value else None

    def check(self):
        _check(load().spa_comm_check(self.h), "spa_comm_check")

    def window_selftest(self, nbytes: int = 1 << 20):
        """NCCL comms, collective: the symmetric-window plumbing check of spa_comm_window_selftest."""
        _check(load().spa_comm_window_selftest(self.h, nbytes), "spa_comm_window_selftest")

    def close(self):
        if self.h:
            load().spa_comm_destroy(self.h)
            self.h = None


class Plan:
    def __init__(self, comm: Comm, B: int, S: int, H: int, D: int, stages: int = 1, n_src: int = 0,
                 pad_heads: bool = False, ring: bool = False, ulysses: int = 0):
        self.comm = comm
        self.shape = Shape(B, S, H, D, stages, n_src, int(bool(pad_heads)), int(bool(ring)), int(ulysses))
        h = ctypes.c_void_p()
        _check(load().spa_plan_create(ctypes.byref(h), comm.h, ctypes.byref(self.shape)), "spa_plan_create")
        self.h = h
        self.B, self.S, self.H, self.D, self.stages = B, S, H, D, stages
        self.n_src = n_src or comm.nranks

    @property
    def workspace_bytes(self) -> int:
        n = ctypes.c_size_t()
        _check(load().spa_plan_workspace_bytes(self.h, ctypes.byref(n)), "spa_plan_workspace_bytes")
        return n.value

    @property
    def stage_split(self):
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(load().spa_plan_stage_split(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
               "spa_plan_stage_split")
        return a.value, b.value, c.value

    def set_option(self, option: int, value: int):
        _check(load().spa_plan_set_option(self.h, option, value), "spa_plan_set_option")

    def set_kv_len(self, kv_len):
        """Key-padding lengths (device int32 tensor [B], kept alive by the caller) or None."""
        self._kv_len = kv_len   # keep the tensor referenced while the plan may read it
        _check(load().spa_plan_set_kv_len(self.h, _ptr(kv_len)), "spa_plan_set_kv_len")

    def last_profile(self) -> Profile:
        p = Profile()
        _check(load().spa_plan_last_profile(self.h, ctypes.byref(p)), "spa_plan_last_profile")
        return p

    @property
    def host_sp_workspace_bytes(self) -> int:
        n = ctypes.c_size_t()
        _check(load().spa_plan_host_sp_workspace_bytes(self.h, ctypes.byref(n)), "spa_plan_host_sp_workspace_bytes")
        return n.value

    @property
    def host_workspace_bytes(self) -> int:
        n = ctypes.c_size_t()
        _check(load().spa_plan_host_workspace_bytes(self.h, ctypes.byref(n)), "spa_plan_host_workspace_bytes")
        return n.value

    def workspace(self, device="cuda"):
        import torch
        return torch.empty(max(self.workspace_bytes, 16), dtype=torch.uint8, device=device)

    # -- P2P plans (CUDA IPC): register the workspace the calls will use
    IPC_HANDLE_BYTES = 72

    def ipc_handle(self, ws) -> bytes:
        buf = ctypes.create_string_buffer(self.IPC_HANDLE_BYTES)
        _check(load().spa_plan_ipc_handle(self.h, _ptr(ws), buf), "spa_plan_ipc_handle")
        return buf.raw

    def ipc_open(self, ws, handles: Sequence[bytes]):
        blob = b"".join(handles)
        assert len(blob) == self.IPC_HANDLE_BYTES * self.comm.nranks
        _check(load().spa_plan_ipc_open(self.h, _ptr(ws), blob), "spa_plan_ipc_open")

    def ipc_setup(self, ws, group=None):
        """Collective: exchange the IPC handles of every rank's ws over torch.distributed and map them."""
        import torch.distributed as dist
        hs = [None] * self.comm.nranks
        dist.all_gather_object(hs, self.ipc_handle(ws), group=group)
        self.ipc_open(ws, hs)
        dist.barrier(group=group)

    # -- NCCL plans on an NCCL symmetric window (peer-memory exchange; spa_plan_window_register)
    def window_setup(self, nbytes: Optional[int] = None, group=None) -> int:
        """Collective: allocate this rank's workspace (nbytes, default workspace_bytes; e.g. qkv_workspace_bytes for
        the fused-projection calls) with NCCL's allocator, register it as a symmetric window and barrier; returns the
        device address to pass as ws (freed by close(), after the plan is destroyed)."""
        import torch.distributed as dist
        n = (max(nbytes if nbytes is not None else self.workspace_bytes, 1) + 4095) // 4096 * 4096
        ptr = ctypes.c_void_p()
        _check(load().spa_mem_alloc(n, ctypes.byref(ptr)), "spa_mem_alloc")
        self._window_ws = ptr.value
        _check(load().spa_plan_window_register(self.h, ctypes.c_void_p(ptr.value)), "spa_plan_window_register")
        if dist.is_available() and dist.is_initialized():
            dist.barrier(group=group)
        return ptr.value

    # -- QKV projection
    def qkv_weight_bytes(self, C: int) -> int:
        n = ctypes.c_size_t()
        _check(load().spa_plan_qkv_weight_bytes(self.h, C, ctypes.byref(n)), "spa_plan_qkv_weight_bytes")
        return n.value

    @property
    def qkv_workspace_bytes(self) -> int:
        n = ctypes.c_size_t()
        _check(load().spa_plan_qkv_workspace_bytes(self.h, ctypes.byref(n)), "spa_plan_qkv_workspace_bytes")
        return n.value

    def qkv_workspace(self, device="cuda"):
        import torch
        return torch.empty(max(self.qkv_workspace_bytes, 16), dtype=torch.uint8, device=device)

    def pack_qkv_weight(self, w, bias=None, stream=None):
        """w: bf16 [3*H*D, C] device tensor (fused nn.Linear weight), bias: fp32 [3*H*D] or None -> packed buffer."""
        import torch
        C = w.shape[1]
        wp = torch.empty(self.qkv_weight_bytes(C), dtype=torch.uint8, device=w.device)
        _check(load().spa_plan_pack_qkv_weight(self.h, C, _ptr(w), _ptr(bias), _ptr(wp), _stream(stream)),
               "spa_plan_pack_qkv_weight")
        return wp

    # -- host-side descriptions (no GPU needed)
    def describe_pack(self, rank: int) -> List[CopyDesc]:
        cap = 3 * self.comm.nranks * max(1, self.H) + 16
        out = (CopyDesc * cap)()
        n = ctypes.c_int()
        _check(load().spa_plan_describe_pack(self.h, rank, out, cap, ctypes.byref(n)), "describe_pack")
        return list(out[:n.value])

    def describe_unpack(self, rank: int) -> List[CopyDesc]:
        cap = self.comm.nranks * max(1, self.H) + 16
        out = (CopyDesc * cap)()
        n = ctypes.c_int()
        _check(load().spa_plan_describe_unpack(self.h, rank, out, cap, ctypes.byref(n)), "describe_unpack")
        return list(out[:n.value])

    def describe_messages(self, stage: int, direction: int, rank: int) -> List[Msg]:
        cap = 4 * self.comm.nranks * self.B * 3 + 16
        out = (Msg * cap)()
        n = ctypes.c_int()
        _check(load().spa_plan_describe_messages(self.h, stage, direction, rank, out, cap, ctypes.byref(n)),
               "describe_messages")
        return list(out[:n.value])

    def describe_ring(self, step: int, rank: int) -> List[Msg]:
        out = (Msg * 8)()
        n = ctypes.c_int()
        _check(load().spa_plan_describe_ring(self.h, step, rank, out, 8, ctypes.byref(n)), "describe_ring")
        return list(out[:n.value])

    def describe_attention(self, stage: int, rank: int) -> AttnDesc:
        d = AttnDesc()
        _check(load().spa_plan_describe_attention(self.h, stage, rank, ctypes.byref(d)), "describe_attention")
        return d

    def close(self):
        if self.h:
            load().spa_plan_destroy(self.h)
            self.h = None
        if getattr(self, "_window_ws", None):
            load().spa_mem_free(ctypes.c_void_p(self._window_ws))
            self._window_ws = None


# ------------------------------------------------------------------ calls (same names as the C ABI)
def spa_attention_fwd(q, k, v, o, B, Sq, Skv, n_heads, D, q_tok_stride, q_batch_stride, kv_tok_stride,
                      kv_batch_stride, o_tok_stride, o_batch_stride, stream=None):
    _check(load().spa_attention_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(o), B, Sq, Skv, n_heads, D, q_tok_stride,
                                    q_batch_stride, kv_tok_stride, kv_batch_stride, o_tok_stride, o_batch_stride,
                                    _stream(stream)), "spa_attention_fwd")


def spa_attention_fwd_masked(q, k, v, o, B, Sq, Skv, n_heads, D, q_tok_stride, q_batch_stride, kv_tok_stride,
                             kv_batch_stride, o_tok_stride, o_batch_stride, kv_len, stream=None):
    _check(load().spa_attention_fwd_masked(_ptr(q), _ptr(k), _ptr(v), _ptr(o), B, Sq, Skv, n_heads, D,
                                           q_tok_stride, q_batch_stride, kv_tok_stride, kv_batch_stride,
                                           o_tok_stride, o_batch_stride, _ptr(kv_len), _stream(stream)),
           "spa_attention_fwd_masked")


def spa_attention_fwd_ex(q, k, v, o, B, Sq, Skv, n_heads, D, q_tok_stride, q_batch_stride, kv_tok_stride,
                         kv_batch_stride, o_tok_stride, o_batch_stride, kv_len=None, out_fp32=0, lse=None, stream=None):
    _check(load().spa_attention_fwd_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(o), B, Sq, Skv, n_heads, D, q_tok_stride,
                                       q_batch_stride, kv_tok_stride, kv_batch_stride, o_tok_stride, o_batch_stride,
                                       _ptr(kv_len), int(out_fp32), _ptr(lse), _stream(stream)), "spa_attention_fwd_ex")


def attention_fp32(q, k, v, kv_len=None, stream=None):
    """Diagnostic single-GPU attention on contiguous bf16 [B, S, H, D]: (fp32 output [B, S, H, D], lse [B, S, H])."""
    import torch
    B, Sq, H, D = q.shape
    Skv = k.shape[1]
    o = torch.empty((B, Sq, H, D), dtype=torch.float32, device=q.device)
    lse = torch.empty((B, Sq, H), dtype=torch.float32, device=q.device)
    spa_attention_fwd_ex(q, k, v, o, B, Sq, Skv, H, D, H * D, Sq * H * D, H * D, Skv * H * D, H * D, Sq * H * D,
                         kv_len, 1, lse, stream)
    return o, lse


def attention(q, k, v, out=None, stream=None, kv_len=None):
    """Single-GPU multi-head attention on contiguous bf16 [B, S, H, D] tensors (all heads).
    kv_len: optional device int32 [B] key-padding lengths (keys t >= kv_len[b] masked)."""
    import torch
    assert q.dtype == torch.bfloat16 and q.is_contiguous() and k.is_contiguous() and v.is_contiguous()
    B, Sq, H, D = q.shape
    Skv = k.shape[1]
    if out is None:
        out = torch.empty_like(q)
    if kv_len is None:
        spa_attention_fwd(q, k, v, out, B, Sq, Skv, H, D, H * D, Sq * H * D, H * D, Skv * H * D, H * D,
                          Sq * H * D, stream)
    else:
        assert kv_len.dtype == torch.int32 and kv_len.is_cuda and kv_len.numel() == B
        spa_attention_fwd_masked(q, k, v, out, B, Sq, Skv, H, D, H * D, Sq * H * D, H * D, Skv * H * D, H * D,
                                 Sq * H * D, kv_len, stream)
    return out


def spa_ulysses_attention(plan: Plan, q, k, v, out, ws, stream=None):
    _check(load().spa_ulysses_attention(plan.h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(ws), _stream(stream)),
           "spa_ulysses_attention")


def spa_pipesp_attention(plan: Plan, q, k, v, out, ws, stream=None):
    _check(load().spa_pipesp_attention(plan.h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(ws), _stream(stream)),
           "spa_pipesp_attention")


def spa_aco_attention(plan: Plan, q, k, v, out, ws, stream=None):
    _check(load().spa_aco_attention(plan.h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(ws), _stream(stream)),
           "spa_aco_attention")


def spa_ulysses_attention_local(plan: Plan, qs, ks, vs, outs, ws, stream=None):
    _check(load().spa_ulysses_attention_local(plan.h, _arr(qs), _arr(ks), _arr(vs), _arr(outs), _ptr(ws),
                                              _stream(stream)), "spa_ulysses_attention_local")


def spa_pipesp_attention_local(plan: Plan, qs, ks, vs, outs, ws, stream=None):
    _check(load().spa_pipesp_attention_local(plan.h, _arr(qs), _arr(ks), _arr(vs), _arr(outs), _ptr(ws),
                                             _stream(stream)), "spa_pipesp_attention_local")


def spa_aco_attention_local(plan: Plan, qs, ks, vs, outs, ws, stream=None):
    _check(load().spa_aco_attention_local(plan.h, _arr(qs), _arr(ks), _arr(vs), _arr(outs), _ptr(ws),
                                          _stream(stream)), "spa_aco_attention_local")


def spa_attention_host(plan: Plan, q, k, v, o, ws, stream=None):
    """q, k, v, o: host (pinned) bf16 [B, S, H, D] tensors; ws: device workspace of plan.host_workspace_bytes."""
    _check(load().spa_attention_host(plan.h, _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(ws), _stream(stream)),
           "spa_attention_host")


def spa_pipesp_attention_hostbuf(plan: Plan, q, k, v, out, ws, stream=None):
    """q, k, v, out: this rank's pinned host bf16 [B, S_r, H, D] (None on Aco co-processor ranks)."""
    _check(load().spa_pipesp_attention_hostbuf(plan.h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(ws),
                                               _stream(stream)), "spa_pipesp_attention_hostbuf")


def spa_pipesp_attention_hostbuf_local(plan: Plan, qs, ks, vs, outs, ws, stream=None):
    _check(load().spa_pipesp_attention_hostbuf_local(plan.h, _arr(qs), _arr(ks), _arr(vs), _arr(outs), _ptr(ws),
                                                     _stream(stream)), "spa_pipesp_attention_hostbuf_local")


def spa_ring_attention(plan: Plan, q, k, v, out, ws, stream=None):
    _check(load().spa_ring_attention(plan.h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(ws), _stream(stream)),
           "spa_ring_attention")


def spa_ring_attention_local(plan: Plan, qs, ks, vs, outs, ws, stream=None):
    _check(load().spa_ring_attention_local(plan.h, _arr(qs), _arr(ks), _arr(vs), _arr(outs), _ptr(ws),
                                           _stream(stream)), "spa_ring_attention_local")


def spa_reshard_seq_to_head(plan: Plan, x, x_head, ws, stream=None):
    _check(load().spa_reshard_seq_to_head(plan.h, _ptr(x), _ptr(x_head), _ptr(ws), _stream(stream)),
           "spa_reshard_seq_to_head")


def spa_reshard_head_to_seq(plan: Plan, x_head, x, ws, stream=None):
    _check(load().spa_reshard_head_to_seq(plan.h, _ptr(x_head), _ptr(x), _ptr(ws), _stream(stream)),
           "spa_reshard_head_to_seq")


def spa_reshard_seq_to_head_local(plan: Plan, xs, x_heads, ws, stream=None):
    _check(load().spa_reshard_seq_to_head_local(plan.h, _arr(xs), _arr(x_heads), _ptr(ws), _stream(stream)),
           "spa_reshard_seq_to_head_local")


def spa_reshard_head_to_seq_local(plan: Plan, x_heads, xs, ws, stream=None):
    _check(load().spa_reshard_head_to_seq_local(plan.h, _arr(x_heads), _arr(xs), _ptr(ws), _stream(stream)),
           "spa_reshard_head_to_seq_local")


def spa_pipesp_qkv_attention(plan: Plan, C: int, x, w_packed, out, ws, stream=None):
    _check(load().spa_pipesp_qkv_attention(plan.h, C, _ptr(x), _ptr(w_packed), _ptr(out), _ptr(ws), _stream(stream)),
           "spa_pipesp_qkv_attention")


def spa_pipesp_qkv_attention_local(plan: Plan, C: int, xs, w_packed, outs, ws, stream=None):
    _check(load().spa_pipesp_qkv_attention_local(plan.h, C, _arr(xs), _ptr(w_packed), _arr(outs), _ptr(ws),
                                                 _stream(stream)), "spa_pipesp_qkv_attention_local")


def spa_qkv_projection(plan: Plan, C: int, rank: int, x, w_packed, q, k, v, stream=None):
    _check(load().spa_qkv_projection(plan.h, C, rank, _ptr(x), _ptr(w_packed), _ptr(q), _ptr(k), _ptr(v),
                                     _stream(stream)), "spa_qkv_projection")
