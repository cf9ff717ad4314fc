"""Python binding of libee_b200.so (include/ee.h) -- argument marshalling only.

Every step of the EE-Tuning exit-head path runs in the CUDA library; this
module converts torch tensors to device pointers, calls the C-ABI functions of
the same names, and raises on a non-OK status.  PyTorch is used for device
memory and streams only.  There is no CPU fallback: if the library or an sm_100
GPU is missing, the calls raise.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libee_b200.so")

EE_OK = 0
STATUS_NAMES = {0: "EE_OK", 1: "EE_ERR_ARG", 2: "EE_ERR_SHAPE", 3: "EE_ERR_ALIGN",
                4: "EE_ERR_VOCAB", 5: "EE_ERR_ARCH", 6: "EE_ERR_STRUCTURE",
                7: "EE_ERR_DIVERGED", 8: "EE_ERR_WORKSPACE", 9: "EE_ERR_CUDA",
                10: "EE_ERR_NCCL", 11: "EE_ERR_UNSUPPORTED", 12: "EE_ERR_PEER"}
ARCH = {"embedding": 0, "norm": 1, "mlp": 2, "layer": 3}
INIT = {"copy": 0, "random": 1}
DTYPE = {torch.bfloat16: 0, torch.float32: 1}
TENSOR_NAMES = ("g_a", "w_gate", "w_up", "w_down", "g_f", "w_out", "g_att", "w_q", "w_k", "w_v",
                "w_o")
EXPORTED = ("ee_workspace_size", "ee_init_heads", "ee_tune_step", "ee_count_valid",
            "ee_adam_update", "ee_sgd_update", "ee_get_status", "ee_lr_at", "ee_last_error",
            "ee_version", "ee_test_gemm", "ee_profile_start", "ee_profile_stop",
            "ee_profile_record", "ee_launch_count", "ee_vp_exit_forward", "ee_vp_vocab_stats",
            "ee_vp_rescale", "ee_vp_vocab_backward", "ee_vp_exit_backward", "ee_exit_infer",
            "ee_backbone_workspace_size", "ee_backbone_forward", "ee_test_attention",
            "ee_normalize_exit", "ee_vp_exit_forward_ag", "ee_vp_vocab_backward_rs",
            "ee_vp_exit_backward_slots", "ee_peer_barrier", "ee_ipc_get_handle", "ee_ipc_open",
            "ee_ipc_close", "ee_dp_shard_layout", "ee_tune_step_rs", "ee_adam_update_sharded",
            "ee_tune_step_adam", "ee_comm_arena_size", "ee_comm_create", "ee_comm_destroy")
MAX_PEERS = 8


class EEError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


class ee_head_config(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("vocab", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("num_exits", ctypes.c_int32), ("arch", ctypes.c_int32),
                ("norm_eps", ctypes.c_float), ("vocab_begin", ctypes.c_int32),
                ("vocab_end", ctypes.c_int32), ("token_weighting", ctypes.c_int32),
                ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("seq_len", ctypes.c_int32), ("rope_theta", ctypes.c_float),
                ("ds_mode", ctypes.c_int32)]


class ee_head_tensors(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in TENSOR_NAMES]


class ee_backbone_config(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("seq_len", ctypes.c_int32), ("norm_eps", ctypes.c_float),
                ("rope_theta", ctypes.c_float)]


LAYER_NAMES = ("g_att", "w_q", "w_k", "w_v", "w_o", "g_mlp", "w_gate", "w_up", "w_down")


class ee_layer_tensors(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in LAYER_NAMES]


AUX_NAMES = ("lse", "loss_tok", "argmax", "conf", "weight_sum")


class ee_step_aux(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in AUX_NAMES]


class ee_peer_set(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("ptr", ctypes.c_void_p * MAX_PEERS)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the CUDA library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -m paper_2402_00518_b200.build` "
                          "or __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    P, I32, I64, F32, SZ = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                            ctypes.c_size_t)
    CFG = ctypes.POINTER(ee_head_config)
    HT = ctypes.POINTER(ee_head_tensors)
    sig = {
        "ee_workspace_size": (I32, [CFG, I64, ctypes.POINTER(SZ)]),
        "ee_init_heads": (I32, [CFG, I32, HT, I32, ctypes.c_uint64, F32, HT, HT, P]),
        "ee_tune_step": (I32, [CFG, ctypes.POINTER(P), I64, P, ctypes.POINTER(F32), HT, HT, I32,
                               P, ctypes.POINTER(ee_step_aux), P, P, SZ, P, P]),
        "ee_comm_arena_size": (I32, [CFG, I32, I32, I64, ctypes.POINTER(SZ)]),
        "ee_comm_create": (I32, [ctypes.POINTER(P), CFG, I32, I32, I32, I64, ctypes.POINTER(P),
                                 SZ]),
        "ee_comm_destroy": (I32, [P]),
        "ee_count_valid": (I32, [P, I64, I32, P, P, SZ, P]),
        "ee_adam_update": (I32, [CFG, HT, HT, HT, HT, HT, F32, F32, F32, F32, F32, I64, F32, P]),
        "ee_sgd_update": (I32, [CFG, HT, HT, HT, HT, F32, F32, F32, P]),
        "ee_get_status": (I32, [P, P, ctypes.POINTER(I32), ctypes.POINTER(I32)]),
        "ee_lr_at": (ctypes.c_double, [I64, I64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double]),
        "ee_last_error": (ctypes.c_char_p, []),
        "ee_version": (ctypes.c_char_p, []),
        "ee_test_gemm": (I32, [I32, I32, P, P, P, I32, I32, I32, I32, P]),
        "ee_normalize_exit": (I32, [CFG, HT, P, P, P]),
        "ee_test_attention": (I32, [P, P, P, P, P, P, P, P, P, P, I64, I32, I32, I32, I32, P]),
        "ee_profile_start": (I32, []),
        "ee_profile_stop": (I32, [ctypes.POINTER(I32)]),
        "ee_profile_record": (I32, [I32, ctypes.c_char_p, I32, ctypes.POINTER(F32),
                                    ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double)]),
        "ee_launch_count": (I64, []),
        "ee_vp_exit_forward": (I32, [CFG, P, I64, I64, HT, P, P, SZ, P]),
        "ee_vp_vocab_stats": (I32, [CFG, P, I64, P, HT, P, P, P, SZ, P]),
        "ee_vp_rescale": (I32, [CFG, I64, P, P, P, SZ, P]),
        "ee_vp_vocab_backward": (I32, [CFG, P, I64, P, P, P, F32, P, HT, HT, I32, P, P,
                                       ctypes.POINTER(ee_step_aux), I32, P, SZ, P]),
        "ee_vp_exit_backward": (I32, [CFG, P, I64, I64, HT, P, HT, I32, P, SZ, P]),
        "ee_vp_exit_forward_ag": (I32, [CFG, P, I64, I64, HT, ctypes.POINTER(ee_peer_set), P, SZ,
                                        P]),
        "ee_vp_vocab_backward_rs": (I32, [CFG, P, I64, P, P, P, F32, P, HT, HT, I32,
                                          ctypes.POINTER(ee_peer_set), P,
                                          ctypes.POINTER(ee_step_aux), I32, P, SZ, P]),
        "ee_vp_exit_backward_slots": (I32, [CFG, P, I64, I64, HT, P, I32, HT, I32,
                                            ctypes.POINTER(ee_peer_set), P, SZ, P]),
        "ee_peer_barrier": (I32, [ctypes.POINTER(ee_peer_set), ctypes.c_uint32, P, P]),
        "ee_tune_step_adam": (I32, [CFG, ctypes.POINTER(P), I64, P, ctypes.POINTER(F32), HT, HT,
                                    HT, HT, F32, F32, F32, F32, F32, I64, F32, P,
                                    ctypes.POINTER(ee_step_aux), P, P, SZ, P]),
        "ee_dp_shard_layout": (I32, [CFG, I32, I32, I32, ctypes.POINTER(I64),
                                     ctypes.POINTER(I64), ctypes.POINTER(I64),
                                     ctypes.POINTER(I64)]),
        "ee_tune_step_rs": (I32, [CFG, ctypes.POINTER(P), I64, P, ctypes.POINTER(F32), HT,
                                  ctypes.POINTER(ee_peer_set), P, ctypes.POINTER(ee_step_aux), P,
                                  P, SZ, P]),
        "ee_adam_update_sharded": (I32, [CFG, I32, I32, ctypes.POINTER(P), HT, HT, HT,
                                         ctypes.POINTER(ee_peer_set), F32, F32, F32, F32, F32,
                                         I64, F32, ctypes.c_uint32, P, P]),
        "ee_ipc_get_handle": (I32, [P, P, ctypes.POINTER(ctypes.c_uint64)]),
        "ee_ipc_open": (I32, [P, ctypes.c_uint64, ctypes.POINTER(P)]),
        "ee_ipc_close": (I32, [P, ctypes.c_uint64]),
        "ee_exit_infer": (I32, [CFG, ctypes.POINTER(P), I64, HT, F32, ctypes.POINTER(P),
                                ctypes.POINTER(P), P, P, SZ, P]),
        "ee_backbone_workspace_size": (I32, [ctypes.POINTER(ee_backbone_config), I64,
                                             ctypes.POINTER(SZ)]),
        "ee_backbone_forward": (I32, [ctypes.POINTER(ee_backbone_config),
                                      ctypes.POINTER(ee_layer_tensors), I32, P, I64,
                                      ctypes.POINTER(I32), I32, ctypes.POINTER(P), P, SZ, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(code: int):
    if code != EE_OK:
        raise EEError(code, _lib.ee_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


WEIGHTING = {"uniform": 0, "confidence": 1, "confidence_sum": 2}
DS_MODE = {"recompute": 0, "stored_p": 1}


def make_config(hidden, vocab, ffn, num_exits, arch, norm_eps=1e-5, vocab_begin=0, vocab_end=None,
                token_weighting="uniform", n_heads=0, n_kv_heads=0, seq_len=0, rope_theta=10000.0,
                ds_mode="recompute"):
    """ee_head_config; n_heads / n_kv_heads / seq_len / rope_theta are the Layer
    exit's attention geometry (n_heads defaults to hidden / 128); ds_mode is
    "recompute" (default: S recomputed for dS, logits never in HBM) or
    "stored_p" (the A24 ablation, include/ee.h ee_ds_mode)."""
    a = ARCH[arch] if isinstance(arch, str) else arch
    if a == ARCH["layer"] and not n_heads:
        n_heads = hidden // 128
    if a == ARCH["layer"] and not n_kv_heads:
        n_kv_heads = n_heads
    return ee_head_config(hidden, vocab, ffn, num_exits, a, norm_eps, vocab_begin,
                          vocab if vocab_end is None else vocab_end,
                          WEIGHTING[token_weighting] if isinstance(token_weighting, str)
                          else token_weighting, n_heads, n_kv_heads, seq_len, rope_theta,
                          DS_MODE[ds_mode] if isinstance(ds_mode, str) else ds_mode)


def heads(list_of_dicts):
    """[{name: tensor}] -> ctypes array of ee_head_tensors (missing names -> NULL)."""
    arr = (ee_head_tensors * len(list_of_dicts))()
    for i, d in enumerate(list_of_dicts):
        for n in TENSOR_NAMES:
            t = d.get(n) if d is not None else None
            setattr(arr[i], n, None if t is None else t.data_ptr())
    return arr


# ---------------------------------------------------------------------------
# thin wrappers with the C-ABI names
# ---------------------------------------------------------------------------

def ee_workspace_size(cfg, n_tokens: int) -> int:
    load()
    out = ctypes.c_size_t(0)
    _check(_lib.ee_workspace_size(ctypes.byref(cfg), int(n_tokens), ctypes.byref(out)))
    return out.value


def ee_init_heads(cfg, init, copy_src, master, operand, seed=0, std=0.02, src_dtype=torch.bfloat16,
                  stream=None):
    load()
    src = heads(copy_src) if copy_src is not None else None
    _check(_lib.ee_init_heads(ctypes.byref(cfg), INIT[init] if isinstance(init, str) else init,
                              src, DTYPE[src_dtype], int(seed), float(std), heads(master),
                              heads(operand), _stream(stream)))


def ee_tune_step(cfg, hidden, targets, exit_weights, params, grads, loss_out, workspace,
                 accumulate=False, aux=None, valid_count=None, stream=None, comm=None):
    """One step over all exits (include/ee.h); comm (a Comm) runs the DP / VP
    step over the communicator's ranks in the same call."""
    load()
    E = cfg.num_exits
    hid = (ctypes.c_void_p * E)(*[h.data_ptr() for h in hidden])
    w = (ctypes.c_float * E)(*[float(a) for a in exit_weights])
    ax = None
    if aux is not None:
        ax = (ee_step_aux * E)()
        for i, d in enumerate(aux):
            for k in AUX_NAMES:
                t = d.get(k)
                setattr(ax[i], k, None if t is None else t.data_ptr())
    n = targets.numel()
    _check(_lib.ee_tune_step(ctypes.byref(cfg), hid, n, _ptr(targets), w, heads(params),
                             heads(grads), int(bool(accumulate)), _ptr(loss_out), ax,
                             _ptr(valid_count), _ptr(workspace), workspace.numel(),
                             None if comm is None else comm.handle, _stream(stream)))


COMM_MODE = {"dp": 0, "vp": 1}


def ee_comm_arena_size(cfg, mode, world, n_local) -> int:
    load()
    b = ctypes.c_size_t(0)
    _check(_lib.ee_comm_arena_size(ctypes.byref(cfg), COMM_MODE[mode], world, n_local,
                                   ctypes.byref(b)))
    return b.value


class Comm:
    """The in-library communicator of one rank (include/ee.h ee_comm_*): a
    zero-filled symmetric arena (torch allocation), the other ranks' arenas
    mapped into this process, and the library handle.  After construction on
    every rank, ee_tune_step(..., comm=c) runs a whole DP / VP step.

    exchange(obj) -> [obj of rank 0, ..., obj of rank world-1] is any host
    transport (store_exchange over a TCPStore, dist.all_gather_object, ...);
    it carries the CUDA IPC handles.  Ranks sharing one process (tests) use
    Comm.local instead."""

    def __init__(self, cfg, mode, world, rank, n_local, exchange=None, device="cuda",
                 _arenas=None):
        load()
        self.mode, self.world, self.rank, self.n_local = mode, world, rank, n_local
        self.bytes = ee_comm_arena_size(cfg, mode, world, n_local)
        self._opened = []
        if _arenas is None:
            self._raw = torch.zeros(self.bytes + 256, dtype=torch.uint8, device=device)
            self.arena = self._raw[(-self._raw.data_ptr()) % 256:][:self.bytes]
            torch.cuda.synchronize(device)     # zero-filled before any peer can write
            mine = ee_ipc_get_handle(self.arena) if world > 1 else None
            allh = exchange(mine) if world > 1 else [mine]
            ptrs = []
            for q in range(world):
                if q == rank:
                    ptrs.append(self.arena.data_ptr())
                else:
                    p = ee_ipc_open(*allh[q])
                    self._opened.append((p, allh[q][1]))
                    ptrs.append(p)
        else:
            self.arena = _arenas[rank]
            ptrs = [a.data_ptr() for a in _arenas]
        arr = (ctypes.c_void_p * world)(*ptrs)
        h = ctypes.c_void_p()
        _check(_lib.ee_comm_create(ctypes.byref(h), ctypes.byref(cfg), COMM_MODE[mode], world,
                                   rank, n_local, arr, self.bytes))
        self.handle = h

    @classmethod
    def local(cls, cfgs, mode, world, n_local, device="cuda"):
        """All ranks' comms inside one process (ranks emulated by threads /
        streams on one GPU): cfgs[r] is rank r's config."""
        b = ee_comm_arena_size(cfgs[0], mode, world, n_local)
        raws = [torch.zeros(b + 256, dtype=torch.uint8, device=device) for _ in range(world)]
        ars = [r[(-r.data_ptr()) % 256:][:b] for r in raws]
        torch.cuda.synchronize(device)
        out = [cls(cfgs[r], mode, world, r, n_local, _arenas=ars) for r in range(world)]
        for c in out:
            c._raws = raws
        return out

    def close(self):
        if self.handle:
            _lib.ee_comm_destroy(self.handle)
            self.handle = None
        for p, off in self._opened:
            ee_ipc_close(p, off)
        self._opened = []


def store_exchange(store, rank: int, world: int, prefix: str):
    """An exchange() for Comm over a torch.distributed Store (e.g. TCPStore):
    no process group needed."""
    import pickle
    n = [0]

    def ex(obj):
        n[0] += 1
        store.set(f"{prefix}/{n[0]}/{rank}", pickle.dumps(obj))
        return [pickle.loads(store.get(f"{prefix}/{n[0]}/{q}")) for q in range(world)]
    return ex


def ee_exit_infer(cfg, hidden, params, threshold, argmax_out, conf_out, workspace,
                  first_exit=None, stream=None):
    """Greedy token + confidence per exit and the first exit reaching
    `threshold`."""
    load()
    E = cfg.num_exits
    n = hidden[0].shape[0] if E else 0
    hid = (ctypes.c_void_p * E)(*[h.data_ptr() for h in hidden])
    am = (ctypes.c_void_p * E)(*[a.data_ptr() for a in argmax_out])
    cf = (ctypes.c_void_p * E)(*[c.data_ptr() for c in conf_out])
    _check(_lib.ee_exit_infer(ctypes.byref(cfg), hid, n, heads(params), float(threshold), am, cf,
                              _ptr(first_exit), _ptr(workspace), workspace.numel(),
                              _stream(stream)))


def make_backbone_config(hidden, n_heads, n_kv_heads, ffn, seq_len, norm_eps=1e-5,
                         rope_theta=10000.0):
    return ee_backbone_config(hidden, n_heads, n_kv_heads, ffn, seq_len, norm_eps, rope_theta)


def ee_backbone_workspace_size(cfg, n_tokens) -> int:
    load()
    out = ctypes.c_size_t(0)
    _check(_lib.ee_backbone_workspace_size(ctypes.byref(cfg), int(n_tokens), ctypes.byref(out)))
    return out.value


def ee_backbone_forward(cfg, layers, x0, exit_after, hidden_out, workspace, stream=None):
    """Frozen backbone partial forward: runs layers 1..max(exit_after)
    on x0 [n x h] bf16 and writes the state after each exit layer."""
    load()
    L = (ee_layer_tensors * len(layers))()
    for i, d in enumerate(layers):
        for n in LAYER_NAMES:
            setattr(L[i], n, d[n].data_ptr())
    E = len(exit_after)
    ex = (ctypes.c_int32 * E)(*[int(e) for e in exit_after])
    ho = (ctypes.c_void_p * E)(*[t.data_ptr() for t in hidden_out])
    _check(_lib.ee_backbone_forward(ctypes.byref(cfg), L, len(layers), _ptr(x0), x0.shape[0], ex,
                                    E, ho, _ptr(workspace), workspace.numel(), _stream(stream)))


def ee_count_valid(targets, vocab, out, workspace, stream=None):
    load()
    _check(_lib.ee_count_valid(_ptr(targets), targets.numel(), int(vocab), _ptr(out),
                               _ptr(workspace), workspace.numel(), _stream(stream)))


def ee_adam_update(cfg, master, operand, grads, m, v, lr, step, beta1=0.9, beta2=0.95, eps=1e-5,
                   weight_decay=0.0, grad_scale=1.0, stream=None):
    load()
    _check(_lib.ee_adam_update(ctypes.byref(cfg), heads(master), heads(operand), heads(grads),
                               heads(m), heads(v), lr, beta1, beta2, eps, weight_decay,
                               int(step), grad_scale, _stream(stream)))


def ee_sgd_update(cfg, master, operand, grads, lr, momentum=0.0, momentum_buf=None,
                  grad_scale=1.0, stream=None):
    load()
    buf = heads(momentum_buf) if momentum_buf is not None else None
    _check(_lib.ee_sgd_update(ctypes.byref(cfg), heads(master), heads(operand), heads(grads), buf,
                              lr, momentum, grad_scale, _stream(stream)))


def ee_get_status(workspace, stream=None):
    load()
    code, idx = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(_lib.ee_get_status(_ptr(workspace), _stream(stream), ctypes.byref(code),
                              ctypes.byref(idx)))
    return code.value, idx.value


def ee_lr_at(it, total, warmup_frac=0.01, lr_max=1e-4, lr_min=1e-5) -> float:
    load()
    return _lib.ee_lr_at(int(it), int(total), warmup_frac, lr_max, lr_min)


def ee_version() -> str:
    load()
    return _lib.ee_version().decode()


def ee_test_gemm(A, B, C, a_kmajor, b_kmajor, M, N, K, accumulate=False, stream=None):
    load()
    _check(_lib.ee_test_gemm(int(a_kmajor), int(b_kmajor), _ptr(A), _ptr(B), _ptr(C), M, N, K,
                             int(bool(accumulate)), _stream(stream)))


def ee_test_attention(q, k, v, o, lse2, seq_len, n_heads, n_kv_heads, dout=None, dq=None,
                      dk=None, dv=None, scratch=None, impl=1, stream=None):
    load()
    _check(_lib.ee_test_attention(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse2), _ptr(dout),
                                  _ptr(dq), _ptr(dk), _ptr(dv), _ptr(scratch), q.shape[0],
                                  seq_len, n_heads, n_kv_heads, int(impl), _stream(stream)))


def ee_normalize_exit(cfg, grads, loss, weight_sum, stream=None):
    """Divide one exit's gradients (dict) and loss (device [1] or None) by the
    device scalar weight_sum (data-parallel confidence weighting)."""
    load()
    _check(_lib.ee_normalize_exit(ctypes.byref(cfg), None if grads is None else heads([grads]),
                                  _ptr(loss), _ptr(weight_sum), _stream(stream)))


def _aux1(aux):
    if aux is None:
        return None
    ax = ee_step_aux()
    for k in AUX_NAMES:
        t = aux.get(k)
        setattr(ax, k, None if t is None else t.data_ptr())
    return ctypes.pointer(ax)


def ee_vp_exit_forward(cfg, hidden, n_all, params, z_out, workspace, stream=None):
    load()
    n_local = 0 if hidden is None else hidden.shape[0]
    _check(_lib.ee_vp_exit_forward(ctypes.byref(cfg), _ptr(hidden), n_local, int(n_all),
                                   heads([params]), _ptr(z_out), _ptr(workspace),
                                   workspace.numel(), _stream(stream)))


def ee_vp_vocab_stats(cfg, z_all, targets_all, params, key_out, sums_out, workspace, stream=None):
    load()
    _check(_lib.ee_vp_vocab_stats(ctypes.byref(cfg), _ptr(z_all), targets_all.numel(),
                                  _ptr(targets_all), heads([params]), _ptr(key_out),
                                  _ptr(sums_out), _ptr(workspace), workspace.numel(),
                                  _stream(stream)))


def ee_vp_rescale(cfg, n_all, key_global, sums, workspace, stream=None):
    load()
    _check(_lib.ee_vp_rescale(ctypes.byref(cfg), int(n_all), _ptr(key_global), _ptr(sums),
                              _ptr(workspace), workspace.numel(), _stream(stream)))


def ee_vp_vocab_backward(cfg, z_all, targets_all, key_global, sums_global, exit_weight,
                         params, grads, dz_partial, loss_out, workspace, valid_count=None,
                         accumulate=False, aux=None, exit_index=0, stream=None):
    load()
    _check(_lib.ee_vp_vocab_backward(ctypes.byref(cfg), _ptr(z_all), targets_all.numel(),
                                     _ptr(targets_all), _ptr(key_global), _ptr(sums_global),
                                     float(exit_weight), _ptr(valid_count), heads([params]),
                                     heads([grads]), int(bool(accumulate)), _ptr(dz_partial),
                                     _ptr(loss_out), _aux1(aux), int(exit_index),
                                     _ptr(workspace), workspace.numel(), _stream(stream)))


def ee_vp_exit_backward(cfg, hidden, n_all, params, dz_local, grads, workspace,
                        accumulate=False, stream=None):
    load()
    n_local = 0 if hidden is None else hidden.shape[0]
    _check(_lib.ee_vp_exit_backward(ctypes.byref(cfg), _ptr(hidden), n_local, int(n_all),
                                    heads([params]), _ptr(dz_local), heads([grads]),
                                    int(bool(accumulate)), _ptr(workspace), workspace.numel(),
                                    _stream(stream)))


def peer_set(rank: int, ptrs) -> ee_peer_set:
    """ee_peer_set from per-rank device pointers (ints or tensors; entry `rank`
    is this process's own buffer)."""
    ptrs = list(ptrs)
    if not 1 <= len(ptrs) <= MAX_PEERS or not 0 <= rank < len(ptrs):
        raise ValueError("bad peer set")
    ps = ee_peer_set()
    ps.rank, ps.world = rank, len(ptrs)
    for q, p in enumerate(ptrs):
        ps.ptr[q] = p.data_ptr() if isinstance(p, torch.Tensor) else int(p)
    return ps


def ee_vp_exit_forward_ag(cfg, hidden, n_all, params, z_peers: ee_peer_set, workspace,
                          stream=None):
    """a1-a4 with the all-gather of z fused into the a4 stores (include/ee.h)."""
    load()
    n_local = 0 if hidden is None else hidden.shape[0]
    _check(_lib.ee_vp_exit_forward_ag(ctypes.byref(cfg), _ptr(hidden), n_local, int(n_all),
                                      heads([params]), ctypes.byref(z_peers), _ptr(workspace),
                                      workspace.numel(), _stream(stream)))


def ee_vp_vocab_backward_rs(cfg, z_all, targets_all, key_global, sums_global, exit_weight,
                            params, grads, dz_slots: ee_peer_set, loss_out, workspace,
                            valid_count=None, accumulate=False, aux=None, exit_index=0,
                            stream=None):
    """a6-a9 with the reduce-scatter of dz fused into the a8 epilogue stores."""
    load()
    _check(_lib.ee_vp_vocab_backward_rs(ctypes.byref(cfg), _ptr(z_all), targets_all.numel(),
                                        _ptr(targets_all), _ptr(key_global), _ptr(sums_global),
                                        float(exit_weight), _ptr(valid_count), heads([params]),
                                        heads([grads]), int(bool(accumulate)),
                                        ctypes.byref(dz_slots), _ptr(loss_out), _aux1(aux),
                                        int(exit_index), _ptr(workspace), workspace.numel(),
                                        _stream(stream)))


def ee_vp_exit_backward_slots(cfg, hidden, n_all, params, dz_slots, n_slots, grads, workspace,
                              accumulate=False, grad_arenas=None, stream=None):
    """a10-a13 with dz = the rank-ordered sum of this rank's n_slots slots;
    grad_arenas (ee_peer_set): the body gradients go to their owners' arenas."""
    load()
    n_local = 0 if hidden is None else hidden.shape[0]
    _check(_lib.ee_vp_exit_backward_slots(ctypes.byref(cfg), _ptr(hidden), n_local, int(n_all),
                                          heads([params]), _ptr(dz_slots), int(n_slots),
                                          None if grads is None else heads([grads]),
                                          int(bool(accumulate)),
                                          None if grad_arenas is None else
                                          ctypes.byref(grad_arenas), _ptr(workspace),
                                          workspace.numel(), _stream(stream)))


def ee_peer_barrier(signals: ee_peer_set, epoch: int, workspace, stream=None):
    load()
    _check(_lib.ee_peer_barrier(ctypes.byref(signals), ctypes.c_uint32(epoch & 0xFFFFFFFF),
                                _ptr(workspace), _stream(stream)))


def ee_tune_step_adam(cfg, hidden, targets, exit_weights, operand, master, m, v, lr, step,
                      loss_out, workspace, beta1=0.9, beta2=0.95, eps=1e-5, weight_decay=0.0,
                      grad_scale=1.0, aux=None, valid_count=None, stream=None):
    """ee_tune_step + ee_adam_update with the update fused into the
    weight-gradient epilogues; no gradient tensors."""
    load()
    E = cfg.num_exits
    hid = (ctypes.c_void_p * E)(*[h.data_ptr() for h in hidden])
    w = (ctypes.c_float * E)(*[float(a) for a in exit_weights])
    ax = None
    if aux is not None:
        ax = (ee_step_aux * E)()
        for i, d in enumerate(aux):
            for k in AUX_NAMES:
                t = d.get(k)
                setattr(ax[i], k, None if t is None else t.data_ptr())
    _check(_lib.ee_tune_step_adam(ctypes.byref(cfg), hid, targets.numel(), _ptr(targets), w,
                                  heads(operand), heads(master), heads(m), heads(v), lr, beta1,
                                  beta2, eps, weight_decay, int(step), grad_scale,
                                  _ptr(loss_out), ax, _ptr(valid_count), _ptr(workspace),
                                  workspace.numel(), _stream(stream)))


def ee_dp_shard_layout(cfg, world: int, rank: int, tensor: str):
    """(row_begin, rows, arena offset in floats, arena total floats) of `rank`'s
    shard of `tensor` (a TENSOR_NAMES entry) under the fused DP path."""
    load()
    out = [ctypes.c_int64() for _ in range(4)]
    _check(_lib.ee_dp_shard_layout(ctypes.byref(cfg), int(world), int(rank),
                                   TENSOR_NAMES.index(tensor), *[ctypes.byref(o) for o in out]))
    return tuple(o.value for o in out)


def ee_tune_step_rs(cfg, hidden, targets, exit_weights, params, arenas, loss_out, workspace,
                    aux=None, valid_count=None, stream=None):
    """ee_tune_step with every gradient row stored into its owner's arena
    (arenas: one ee_peer_set per exit)."""
    load()
    E = cfg.num_exits
    hid = (ctypes.c_void_p * E)(*[h.data_ptr() for h in hidden])
    w = (ctypes.c_float * E)(*[float(a) for a in exit_weights])
    ar = (ee_peer_set * E)(*arenas)
    ax = None
    if aux is not None:
        ax = (ee_step_aux * E)()
        for i, d in enumerate(aux):
            for k in AUX_NAMES:
                t = d.get(k)
                setattr(ax[i], k, None if t is None else t.data_ptr())
    _check(_lib.ee_tune_step_rs(ctypes.byref(cfg), hid, targets.numel(), _ptr(targets), w,
                                heads(params), ar, _ptr(loss_out), ax, _ptr(valid_count),
                                _ptr(workspace), workspace.numel(), _stream(stream)))


def ee_adam_update_sharded(cfg, world, rank, arenas_local, master_shard, m_shard, v_shard,
                           operand_sets, lr, step, beta1=0.9, beta2=0.95, eps=1e-5,
                           weight_decay=0.0, grad_scale=1.0, tensors=None, grad_divisor=None,
                           stream=None):
    """Sharded Adam + operand all-gather; operand_sets: per exit a dict
    {name: ee_peer_set of every rank's operand tensor}."""
    load()
    E = cfg.num_exits
    ar = (ctypes.c_void_p * E)(*[a.data_ptr() for a in arenas_local])
    ops = (ee_peer_set * (E * len(TENSOR_NAMES)))()
    for i, d in enumerate(operand_sets):
        for k, ps in d.items():
            ops[i * len(TENSOR_NAMES) + TENSOR_NAMES.index(k)] = ps
    _check(_lib.ee_adam_update_sharded(ctypes.byref(cfg), int(world), int(rank), ar,
                                       heads(master_shard), heads(m_shard), heads(v_shard), ops,
                                       lr, beta1, beta2, eps, weight_decay, int(step), grad_scale,
                                       ctypes.c_uint32(0 if tensors is None else
                                                       sum(1 << TENSOR_NAMES.index(k)
                                                           for k in tensors)),
                                       _ptr(grad_divisor), _stream(stream)))


def ee_ipc_get_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t inside it)."""
    load()
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    _check(_lib.ee_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)))
    return h.raw, off.value


def ee_ipc_open(handle: bytes, offset: int) -> int:
    load()
    p = ctypes.c_void_p()
    _check(_lib.ee_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.c_uint64(offset),
                            ctypes.byref(p)))
    return p.value


def ee_ipc_close(ptr: int, offset: int):
    load()
    _check(_lib.ee_ipc_close(ctypes.c_void_p(ptr), ctypes.c_uint64(offset)))


def ee_profile_start():
    load()
    _check(_lib.ee_profile_start())


def ee_profile_stop():
    """Stop recording; returns [(name, ms, flops_exec, flops_alg, bytes)] per launch."""
    load()
    n = ctypes.c_int32(0)
    _check(_lib.ee_profile_stop(ctypes.byref(n)))
    out = []
    buf = ctypes.create_string_buffer(64)
    ms = ctypes.c_float(0)
    fe, fa, by = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
    for i in range(n.value):
        _check(_lib.ee_profile_record(i, buf, 64, ctypes.byref(ms), ctypes.byref(fe),
                                      ctypes.byref(fa), ctypes.byref(by)))
        out.append((buf.value.decode(), ms.value, fe.value, fa.value, by.value))
    return out


def ee_launch_count() -> int:
    load()
    return int(_lib.ee_launch_count())


# ---------------------------------------------------------------------------
# ExitHeads: parameter store + optimizer state + workspace (torch allocations)
# ---------------------------------------------------------------------------

def tensor_shapes(hidden, vocab, ffn, arch, n_kv_heads=0):
    """Parameter shapes of one exit; `vocab` = rows of W_out held (a shard under VP)."""
    s = {"w_out": (vocab, hidden)}
    if arch != "embedding":
        s["g_f"] = (hidden,)
    if arch in ("mlp", "layer"):
        s.update(g_a=(hidden,), w_gate=(ffn, hidden), w_up=(ffn, hidden), w_down=(hidden, ffn))
    if arch == "layer":
        hkv = 128 * (n_kv_heads or hidden // 128)
        s.update(g_att=(hidden,), w_q=(hidden, hidden), w_k=(hkv, hidden), w_v=(hkv, hidden),
                 w_o=(hidden, hidden))
    return s


@dataclass
class HeadSpec:
    hidden: int
    vocab: int
    ffn: int
    num_exits: int
    arch: str
    norm_eps: float = 1e-5
    vocab_begin: int = 0          # vocab-parallel shard of W_out rows [begin, end)
    vocab_end: int | None = None
    token_weighting: str = "uniform"   # or "confidence"
    n_heads: int = 0              # Layer exits: attention geometry (default hidden / 128)
    n_kv_heads: int = 0           # (default n_heads: no GQA)
    seq_len: int = 0
    rope_theta: float = 10000.0
    ds_mode: str = "recompute"    # or "stored_p" (A24 ablation)

    def attn_kwargs(self):
        """make_config keywords beyond the shapes: attention geometry and ds_mode."""
        return dict(n_heads=self.n_heads, n_kv_heads=self.n_kv_heads, seq_len=self.seq_len,
                    rope_theta=self.rope_theta, ds_mode=self.ds_mode)


class HostStager:
    """Streams per-exit hidden states from pinned host memory to the device
    for the host-input step APIs (ExitHeads.step_host, ShardedDPHeads.step
    with hidden_host): exit i + 1's copy runs on a copy stream while exit i
    computes, through two device staging buffers ordered by events.

    Protocol per step: tg = begin(hidden_host, targets_host, st); then for each
    exit i: buf = get(i, st) (stream st waits for exit i's copy and exit
    i + 1's copy is issued), launch exit i's work on st reading buf, release(i,
    st).  The buffers are sized once (max_tokens rows) and never reallocated;
    the copy stream waits for the allocating stream before its first write, so
    blocks the caching allocator recycled from work still queued on that
    stream are not overwritten early."""

    def __init__(self, max_tokens: int, hidden: int, device):
        st = torch.cuda.current_stream(device)
        self.bufs = [torch.empty(max_tokens, hidden, dtype=torch.bfloat16, device=device)
                     for _ in range(2)]
        self.tg = torch.empty(max_tokens, dtype=torch.int32, device=device)
        self.cs = torch.cuda.Stream(device)
        self.cs.wait_stream(st)
        self.copied = [torch.cuda.Event(), torch.cuda.Event()]
        self.free = [torch.cuda.Event(), torch.cuda.Event()]
        self.used = [False, False]
        self.src = None

    def _stage(self, i):
        b = i % 2
        with torch.cuda.stream(self.cs):
            if self.used[b]:         # the previous reader of buffer b (this or the last call)
                self.cs.wait_event(self.free[b])
            self.bufs[b][:self.n].copy_(self.src[i], non_blocking=True)
            self.copied[b].record(self.cs)

    def begin(self, hidden_host, targets_host, st):
        self.src = hidden_host
        self.n = hidden_host[0].shape[0]
        tg = self.tg[:self.n]
        tg.copy_(targets_host, non_blocking=True)   # on st: ordered after st's earlier readers
        self._stage(0)
        return tg

    def get(self, i, st):
        if i + 1 < len(self.src):
            self._stage(i + 1)
        st.wait_event(self.copied[i % 2])
        return self.bufs[i % 2][:self.n]

    def release(self, i, st):
        self.free[i % 2].record(st)
        self.used[i % 2] = True


class ExitHeads:
    """The exit-head parameter store of one EE-Tuning run on one GPU.

    Holds, per exit, the fp32 master parameters, the bf16 operand copies of the
    matrices, fp32 gradients and Adam moments (exits only), and the
    step workspace.  All compute goes through the C-ABI above.
    """

    def __init__(self, spec: HeadSpec, max_tokens: int, device="cuda", adam=True,
                 grad_buffers: int | None = None):
        """grad_buffers = k < num_exits: exits share k fp32 gradient buffers
        (exit i uses buffer i % k), for the per-exit update schedule
        (step_per_exit): "forward, backward, and parameter update for each
        early-exit layer, without any dependency between early exits".
        At the 70B shape with 8 exits this saves 27 GB."""
        load()
        self.spec = spec
        ve = spec.vocab if spec.vocab_end is None else spec.vocab_end
        self.cfg = make_config(spec.hidden, spec.vocab, spec.ffn, spec.num_exits, spec.arch,
                               spec.norm_eps, spec.vocab_begin, ve, spec.token_weighting,
                               **spec.attn_kwargs())
        shapes = tensor_shapes(spec.hidden, ve - spec.vocab_begin, spec.ffn, spec.arch,
                               self.cfg.n_kv_heads)
        dev = torch.device(device)
        E = spec.num_exits

        def alloc(dtype_for):
            return [{k: torch.zeros(s, dtype=dtype_for(k), device=dev) for k, s in shapes.items()}
                    for _ in range(E)]

        f32 = lambda k: torch.float32
        self.master = alloc(f32)
        # operand copies: bf16 matrices; gains alias the fp32 masters
        self.operand = [{k: (m[k] if k.startswith("g_") else
                             torch.zeros(shapes[k], dtype=torch.bfloat16, device=dev))
                         for k in shapes} for m in self.master]
        k = E if grad_buffers is None else max(1, min(int(grad_buffers), E))
        pool = [{n: torch.zeros(sh, dtype=torch.float32, device=dev) for n, sh in shapes.items()}
                for _ in range(k)]
        self.grad_buffers = k
        self.grads = [pool[i % k] for i in range(E)]
        self.exit_cfg = make_config(spec.hidden, spec.vocab, spec.ffn, 1, spec.arch,
                                    spec.norm_eps, spec.vocab_begin, ve, spec.token_weighting,
                                    **spec.attn_kwargs())
        self.m = alloc(f32) if adam else None
        self.v = alloc(f32) if adam else None
        self.step_count = 0
        self.max_tokens = int(max_tokens)
        ws = ee_workspace_size(self.cfg, self.max_tokens)
        self.workspace = torch.zeros(ws, dtype=torch.uint8, device=dev)
        self.loss = torch.zeros(E, dtype=torch.float32, device=dev)

    def init(self, mode="copy", copy_src=None, seed=0, std=0.02, src_dtype=torch.bfloat16):
        ee_init_heads(self.cfg, mode, copy_src, self.master, self.operand, seed=seed, std=std,
                      src_dtype=src_dtype)

    def step(self, hidden, targets, exit_weights=None, accumulate=False, aux=None,
             valid_count=None):
        if targets.numel() > self.max_tokens:
            raise ValueError("more tokens than the workspace was sized for")
        self.join()
        w = exit_weights if exit_weights is not None else [1.0] * self.spec.num_exits
        ee_tune_step(self.cfg, hidden, targets, w, self.operand, self.grads, self.loss,
                     self.workspace, accumulate=accumulate, aux=aux, valid_count=valid_count)
        return self.loss

    def infer(self, hidden, threshold):
        """Greedy token, confidence per exit and the first exit reaching
        `threshold`.  Returns (argmax [E] list, conf [E] list, first)."""
        self.join()
        n = hidden[0].shape[0]
        dev = self.loss.device
        am = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(self.spec.num_exits)]
        cf = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(self.spec.num_exits)]
        first = torch.empty(n, dtype=torch.int32, device=dev)
        ee_exit_infer(self.cfg, hidden, self.operand, threshold, am, cf, self.workspace, first)
        return am, cf, first

    def adam(self, lr, beta1=0.9, beta2=0.95, eps=1e-5, weight_decay=0.0, grad_scale=1.0):
        if self.grad_buffers < self.spec.num_exits:
            raise RuntimeError("shared gradient buffers: use step_per_exit()")
        self.join()
        self.step_count += 1
        ee_adam_update(self.cfg, self.master, self.operand, self.grads, self.m, self.v, lr,
                       self.step_count, beta1, beta2, eps, weight_decay, grad_scale)

    # ---- Adam overlapped with the next exit (side stream) -------------------
    def _adam_side(self):
        if getattr(self, "_side", None) is None:
            dev = self.loss.device
            self._side = torch.cuda.Stream(dev)
            self._adam_done = [None] * self.spec.num_exits   # exit i's operand updated
            self._buf_done = [None] * self.grad_buffers      # gradient buffer free again
        return self._side

    def _before_tune(self, i, st):
        """Stream `st` may run exit i's step once exit i's previous Adam (which
        writes its operand) and the Adam that last read i's gradient buffer
        are done."""
        for ev in (self._adam_done[i], self._buf_done[i % self.grad_buffers]):
            if ev is not None:
                st.wait_event(ev)

    def _adam_async(self, i, lr, st, beta1=0.9, beta2=0.95, eps=1e-5, weight_decay=0.0,
                    grad_scale=1.0):
        side = self._side
        ev = torch.cuda.Event()
        ev.record(st)
        side.wait_event(ev)
        ee_adam_update(self.exit_cfg, self.master[i:i + 1], self.operand[i:i + 1],
                       self.grads[i:i + 1], self.m[i:i + 1], self.v[i:i + 1], lr,
                       self.step_count, beta1, beta2, eps, weight_decay, grad_scale, stream=side)
        done = torch.cuda.Event()
        done.record(side)
        self._adam_done[i] = done
        self._buf_done[i % self.grad_buffers] = done

    def step_overlapped(self, hidden, targets, lr, exit_weights=None, valid_count=None,
                        beta1=0.9, beta2=0.95, eps=1e-5, weight_decay=0.0, grad_scale=1.0):
        """One step exit by exit with each exit's Adam on a side stream,
        overlapping the next exit's GEMMs (and, across steps, the next step):
        exit i's next tune waits only for exit i's Adam.  Same results as
        step() + adam() (the same kernels on the same data).  Call join()
        before reading parameters or timing."""
        E = self.spec.num_exits
        w = exit_weights if exit_weights is not None else [1.0] * E
        st = torch.cuda.current_stream(self.loss.device)
        self._adam_side()
        self.step_count += 1
        for i in range(E):
            self._before_tune(i, st)
            ee_tune_step(self.exit_cfg, hidden[i:i + 1], targets, w[i:i + 1],
                         self.operand[i:i + 1], self.grads[i:i + 1], self.loss[i:i + 1],
                         self.workspace, valid_count=valid_count)
            self._adam_async(i, lr, st, beta1, beta2, eps, weight_decay, grad_scale)
        return self.loss

    def join(self, stream=None):
        """Make `stream` (default: current) wait for the side-stream updates."""
        if getattr(self, "_side", None) is not None:
            (stream or torch.cuda.current_stream(self.loss.device)).wait_stream(self._side)

    def step_adam(self, hidden, targets, lr, exit_weights=None, beta1=0.9, beta2=0.95,
                  eps=1e-5, weight_decay=0.0, grad_scale=1.0):
        """step() + adam() in one call, the update fused into the weight-gradient
        epilogues (ee_tune_step_adam).  self.grads are not written."""
        if targets.numel() > self.max_tokens:
            raise ValueError("more tokens than the workspace was sized for")
        w = exit_weights if exit_weights is not None else [1.0] * self.spec.num_exits
        self.join()
        self.step_count += 1
        ee_tune_step_adam(self.cfg, hidden, targets, w, self.operand, self.master, self.m, self.v,
                          lr, self.step_count, self.loss, self.workspace, beta1, beta2, eps,
                          weight_decay, grad_scale)
        return self.loss

    def adam_exit(self, i, lr, step, beta1=0.9, beta2=0.95, eps=1e-5, weight_decay=0.0,
                  grad_scale=1.0):
        ee_adam_update(self.exit_cfg, self.master[i:i + 1], self.operand[i:i + 1],
                       self.grads[i:i + 1], self.m[i:i + 1], self.v[i:i + 1], lr, step, beta1,
                       beta2, eps, weight_decay, grad_scale)

    def step_host(self, hidden_host, targets_host, exit_weights=None, lr=None,
                  fused_adam=False):
        """One tuning step with the cached hidden states in pinned HOST memory
        (the usual place for them: 4.3 GB per step at the 70B shape).  Exit
        i + 1's hidden states are copied host-to-device on a side stream while
        exit i computes (HostStager: two device staging buffers, event-ordered),
        so the PCIe/C2C transfer hides under the exit's GEMMs.  Same results as
        step() on device copies of the same bytes.  With lr given, each exit is
        updated right after its backward: Adam on a side stream overlapping the
        next exit (= step_overlapped(); call join() before reading parameters),
        or fused into the backward's epilogues (fused_adam; = step_adam()).
        Returns the device losses."""
        E = self.spec.num_exits
        n = hidden_host[0].shape[0]
        if n > self.max_tokens:
            raise ValueError("more tokens than the workspace was sized for")
        dev = self.loss.device
        st = torch.cuda.current_stream(dev)
        if getattr(self, "_stager", None) is None:
            self._stager = HostStager(self.max_tokens, self.spec.hidden, dev)
        w = exit_weights if exit_weights is not None else [1.0] * E
        overlap = lr is not None and not fused_adam
        if overlap:
            self._adam_side()
        else:
            self.join()
        if lr is not None:
            self.step_count += 1
        tg = self._stager.begin(hidden_host, targets_host, st)
        for i in range(E):
            buf = self._stager.get(i, st)
            if lr is None or overlap:
                if overlap:
                    self._before_tune(i, st)
                ee_tune_step(self.exit_cfg, [buf], tg, w[i:i + 1], self.operand[i:i + 1],
                             self.grads[i:i + 1], self.loss[i:i + 1], self.workspace)
                if overlap:
                    self._adam_async(i, lr, st)
            else:
                ee_tune_step_adam(self.exit_cfg, [buf], tg, w[i:i + 1],
                                  self.operand[i:i + 1], self.master[i:i + 1], self.m[i:i + 1],
                                  self.v[i:i + 1], lr, self.step_count, self.loss[i:i + 1],
                                  self.workspace)
            self._stager.release(i, st)
        return self.loss

    def step_per_exit(self, hidden, targets, lr, exit_weights=None, valid_count=None,
                      reduce_grads=None):
        """One step exit by exit: tune exit i, (optionally) reduce its gradients,
        Adam on exit i.  With k gradient buffers, exit i's update is
        deferred until exit i + k - 1 has been launched, so a reduction issued
        by reduce_grads(i) (returning async handles) overlaps the next exits'
        compute.  Returns the per-exit losses."""
        E = self.spec.num_exits
        k = self.grad_buffers
        w = exit_weights if exit_weights is not None else [1.0] * E
        self.join()
        self.step_count += 1
        pending = {}

        def finish(j):
            for h in pending.pop(j, []):
                h.wait()
            self.adam_exit(j, lr, self.step_count)

        for i in range(E):
            if i - k >= 0:
                finish(i - k)
            ee_tune_step(self.exit_cfg, hidden[i:i + 1], targets, w[i:i + 1],
                         self.operand[i:i + 1], self.grads[i:i + 1], self.loss[i:i + 1],
                         self.workspace, valid_count=valid_count)
            if reduce_grads is not None:
                pending[i] = reduce_grads(i) or []
        for j in range(max(0, E - k), E):
            finish(j)
        return self.loss

    def status(self):
        return ee_get_status(self.workspace)
