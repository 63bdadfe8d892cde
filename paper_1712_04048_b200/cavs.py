"""Thin ctypes binding of the C-ABI in include/cavs.h (argument marshalling only).

Every step of the hot path runs inside libcavs.so (hand-written CUDA for sm_100a);
this module only converts tensors to pointers.  PyTorch is used for device memory
(the workspace and the caller's arrays) and for the CUDA stream — plumbing only.
There is no CPU fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcavs.so")

TREE_LSTM, TREE_FC = 0, 1
FP32, BF16 = 0, 1
CELLS = {"tree_lstm": TREE_LSTM, "tree_fc": TREE_FC}
PRECISIONS = {"fp32": FP32, "bf16": BF16}
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_ARITY", 3: "E_CYCLE", 4: "E_FANOUT", 5: "E_STATE",
          6: "E_CAPACITY", 7: "E_CUDA", 8: "E_UNSUPPORTED"}


class CavsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class _Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("cell", "N", "h", "d", "precision", "max_graphs", "max_vertices", "max_x")]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1712_04048_b200/build.py` or `__graft_entry__.build()` "
                          "(there is no fallback path)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, SZ, S = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_int
    sig = {
        "cavs_param_count": (SZ, [I32, I32, I32, I32]),
        "cavs_create": (S, [ctypes.POINTER(_Desc), ctypes.c_int, P, ctypes.POINTER(P)]),
        "cavs_set_stream": (S, [P, P]),
        "cavs_workspace_bytes": (SZ, [P]),
        "cavs_set_workspace": (S, [P, P, SZ]),
        "cavs_load_graphs": (S, [P, I32, I32, I32, P, P, P, ctypes.c_int]),
        "cavs_schedule": (S, [P, ctypes.POINTER(I32)]),
        "cavs_get_schedule": (S, [P, P, P, P]),
        "cavs_forward": (S, [P, P, I32, P, P, P]),
        "cavs_forward_inference": (S, [P, P, I32, P, P, P]),
        "cavs_backward": (S, [P, P, P, P]),
        "cavs_train_step_host": (S, [P, I32, I32, I32, P, P, P, P, I32, P, P, P, P, P, P]),
        "cavs_kernel_launches": (I64, [P]),
        "cavs_sync": (S, [P]),
        "cavs_set_grad_event": (S, [P, P]),
        "cavs_softmax_xent": (S, [P, I32, I32, P, P, P, ctypes.c_float, P]),
        "cavs_train_step_host_async": (S, [P, I32, I32, I32, P, P, P, P, I32, P, P, I32, P, P, P]),
        "cavs_set_sync_free": (S, [P, ctypes.c_int]),
        "cavs_last_error": (ctypes.c_char_p, [P]),
        "cavs_path_info": (ctypes.c_char_p, [P]),
        "cavs_profile": (S, [P, ctypes.c_int]),
        "cavs_profile_read": (S, [P, I32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)]),
        "cavs_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name, None)
        if f is None:                      # an older library build (A/B runs); tests check the exports
            continue
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTS = ["cavs_param_count", "cavs_create", "cavs_set_stream", "cavs_workspace_bytes",
           "cavs_set_workspace", "cavs_load_graphs", "cavs_schedule", "cavs_get_schedule",
           "cavs_forward", "cavs_forward_inference", "cavs_backward", "cavs_train_step_host", "cavs_kernel_launches", "cavs_sync", "cavs_set_grad_event", "cavs_softmax_xent", "cavs_train_step_host_async", "cavs_set_sync_free",
           "cavs_last_error", "cavs_path_info", "cavs_destroy", "cavs_profile", "cavs_profile_read"]
PHASES = ["schedule", "prep", "xproj", "fwd_levels", "bwd_roots", "bwd_levels", "lazy", "dx", "reduce"]


def lib():
    return _lib


def param_count(cell, N, h, d) -> int:
    return int(_lib.cavs_param_count(CELLS.get(cell, cell), N, h, d))


def _ptr(a, kind=None, device=None, host_ok=False):
    """Pointer of a C-contiguous numpy array or torch tensor.  `kind` in {"i32", "f32"} checks
    the element type (int64 index arrays would be read as int32 garbage); `device` requires a
    CUDA tensor on that device (host_ok: numpy / CPU tensors allowed, e.g. the *_host calls)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        if kind and a.dtype != (np.int32 if kind == "i32" else np.float32):
            raise TypeError(f"expected {kind}, got numpy {a.dtype}")
        if device is not None and not host_ok:
            raise TypeError("expected a CUDA tensor, got a numpy array")
        return a.ctypes.data
    import torch
    if not a.is_contiguous():
        raise ValueError("tensors must be contiguous")
    if kind and a.dtype != (torch.int32 if kind == "i32" else torch.float32):
        raise TypeError(f"expected {kind}, got {a.dtype}")
    if device is not None:
        if a.is_cuda:
            if a.device != device:
                raise ValueError(f"tensor on {a.device}, context on {device}")
        elif not host_ok:
            raise TypeError("expected a CUDA tensor on the context's device, got a CPU tensor")
    return a.data_ptr()


def softmax_xent(logits, target, dlogits=None, loss=None, scale=1.0, stream=None):
    """cavs_softmax_xent: per-row loss and scale * (softmax - onehot) (in place when dlogits is logits).
    logits [M, vocab] fp32 CUDA, target [M] int32 CUDA (< 0: no loss).  Returns (loss [M], dlogits)."""
    import torch
    M, vocab = int(logits.shape[0]), int(logits.shape[1])
    dev = logits.device
    if dlogits is None:
        dlogits = torch.empty_like(logits)
    if loss is None:
        loss = torch.empty(M, dtype=torch.float32, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    st_code = _lib.cavs_softmax_xent(_ptr(logits, "f32", dev), M, vocab, _ptr(target, "i32", dev), _ptr(loss, "f32", dev),
                                     _ptr(dlogits, "f32", dev), float(scale), ctypes.c_void_p(st.cuda_stream))
    if st_code != 0:
        raise CavsError(st_code, "cavs_softmax_xent failed")
    return loss, dlogits


class Context:
    """One engine instance: F fixed at creation (cell, N, h, d, precision), capacities fixed."""

    def __init__(self, cell, N, h, d, precision="fp32", max_graphs=256, max_vertices=1 << 16,
                 max_x=None, device=0, stream=None):
        import torch
        self._torch = torch
        self.cell, self.N, self.h, self.d = cell, N, h, d
        self.precision = precision
        self.device = torch.device("cuda", device)
        desc = _Desc(CELLS.get(cell, cell), N, h, d, PRECISIONS.get(precision, precision), max_graphs,
                     max_vertices, max_vertices if max_x is None else max_x)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        out = ctypes.c_void_p()
        st = _lib.cavs_create(ctypes.byref(desc), device, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(out))
        if st != 0:
            raise CavsError(st, "cavs_create failed")
        self._ctx = out
        nbytes = int(_lib.cavs_workspace_bytes(self._ctx))
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        self._ws_off, self._ws_bytes = aligned - base, nbytes
        self._check(_lib.cavs_set_workspace(self._ctx, ctypes.c_void_p(aligned), nbytes))
        self.P = param_count(cell, N, h, d)
        self.V = 0
        self.T = 0

    def _check(self, st):
        if st != 0:
            raise CavsError(st, (_lib.cavs_last_error(self._ctx) or b"").decode())

    def set_stream(self, stream):
        self.stream = stream
        self._check(_lib.cavs_set_stream(self._ctx, ctypes.c_void_p(stream.cuda_stream)))

    @property
    def launches(self) -> int:
        return int(_lib.cavs_kernel_launches(self._ctx))

    def path_info(self) -> str:
        """Which kernel path runs the batching tasks (e.g. the persistent level kernel)."""
        return (_lib.cavs_path_info(self._ctx) or b"").decode()

    def profile(self, enable: bool = True):
        """Reset the per-phase accumulators and (de)activate phase timing."""
        self._check(_lib.cavs_profile(self._ctx, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{phase: dict(ms, flops, bytes, launches)} accumulated since profile(True)."""
        out = {}
        for i, name in enumerate(PHASES):
            ms, fl, by = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            ln = ctypes.c_int64()
            self._check(_lib.cavs_profile_read(self._ctx, i, ctypes.byref(ms), ctypes.byref(fl),
                                               ctypes.byref(by), ctypes.byref(ln)))
            out[name] = dict(ms=ms.value, flops=fl.value, bytes=by.value, launches=int(ln.value))
        return out

    def load_graphs(self, graph_ptr, child_ptr, child_idx):
        """CSR child lists per instance; numpy (host) or torch CUDA int32 arrays."""
        on_dev = not isinstance(graph_ptr, np.ndarray)
        K = int(graph_ptr.shape[0]) - 1
        V = int(child_ptr.shape[0]) - 1
        E = int(child_idx.shape[0])
        self._keep = (graph_ptr, child_ptr, child_idx)
        dev = self.device if on_dev else None
        self._check(_lib.cavs_load_graphs(self._ctx, K, V, E, _ptr(graph_ptr, "i32", dev), _ptr(child_ptr, "i32", dev),
                                          _ptr(child_idx, "i32", dev) if E else None, 1 if on_dev else 0))
        self.V, self.K = V, K

    def schedule(self, wait: bool = True):
        """Algorithm 1's task partition.  wait=True returns T (and raises on invalid graphs);
        wait=False only enqueues — T and validation errors surface at the next forward()."""
        if not wait:
            self._check(_lib.cavs_schedule(self._ctx, None))
            self.T = None
            return None
        T = ctypes.c_int32()
        self._check(_lib.cavs_schedule(self._ctx, ctypes.byref(T)))
        self.T = int(T.value)
        return self.T

    def get_schedule(self):
        level = np.empty(self.V, np.int32)
        level_ptr = np.empty(self.T + 1, np.int32)
        order = np.empty(self.V, np.int32)
        self._check(_lib.cavs_get_schedule(self._ctx, level.ctypes.data, level_ptr.ctypes.data, order.ctypes.data))
        return level, level_ptr, order

    def forward(self, params, x, x_row, h_out=None):
        torch = self._torch
        if h_out is None:
            h_out = torch.empty(self.V, self.h, dtype=torch.float32, device=self.device)
        self._fwd_keep = (params, x, x_row, h_out)
        dv = self.device
        self._check(_lib.cavs_forward(self._ctx, _ptr(params, "f32", dv), int(x.shape[0]), _ptr(x, "f32", dv),
                                      _ptr(x_row, "i32", dv), _ptr(h_out, "f32", dv)))
        return h_out

    def forward_inference(self, params, x, x_row, h_out=None):
        """Inference-only forward: same h_out, no activations saved (backward needs forward())."""
        torch = self._torch
        if h_out is None:
            h_out = torch.empty(self.V, self.h, dtype=torch.float32, device=self.device)
        self._fwd_keep = (params, x, x_row, h_out)
        dv = self.device
        self._check(_lib.cavs_forward_inference(self._ctx, _ptr(params, "f32", dv), int(x.shape[0]),
                                                _ptr(x, "f32", dv), _ptr(x_row, "i32", dv), _ptr(h_out, "f32", dv)))
        return h_out

    def backward(self, dh_out, dparams=None, dx=None, want_dx=True):
        torch = self._torch
        if dparams is None:
            dparams = torch.empty(self.P, dtype=torch.float32, device=self.device)
        if dx is None and want_dx:
            x = self._fwd_keep[1]
            dx = torch.empty(x.shape[0], self.d, dtype=torch.float32, device=self.device)
        self._bwd_keep = (dh_out, dparams, dx)
        dv = self.device
        self._check(_lib.cavs_backward(self._ctx, _ptr(dh_out, "f32", dv), _ptr(dparams, "f32", dv),
                                       _ptr(dx, "f32", dv)))
        return dparams, dx

    def set_grad_event(self, event):
        """cavs_set_grad_event: `event` (torch.cuda.Event or None) is recorded by every later backward
        once the weight blocks of dparams are final (before dX and db)."""
        self._grad_event = event
        ptr = None
        if event is not None:
            event.record(self.stream)                    # materialise the cudaEvent_t
            ptr = event.cuda_event
        self._check(_lib.cavs_set_grad_event(self._ctx, ptr))

    def set_sync_free(self, on=True):
        """cavs_set_sync_free: schedule / forward / backward never wait on the host (graph-capturable)."""
        self._check(_lib.cavs_set_sync_free(self._ctx, 1 if on else 0))

    def sync(self):
        """Wait for the context's stream; raises on deferred device-side input errors (cavs_sync)."""
        self._check(_lib.cavs_sync(self._ctx))

    def train_step_host(self, graph_ptr, child_ptr, child_idx, params, x, x_row, dh_out,
                        dparams, dx=None, h_out=None):
        """Whole step from HOST arrays (numpy or pinned CPU tensors); synchronous."""
        K = int(graph_ptr.shape[0]) - 1
        V = int(child_ptr.shape[0]) - 1
        E = int(child_idx.shape[0])
        H = dict(device=self.device, host_ok=True)
        self._check(_lib.cavs_train_step_host(
            self._ctx, K, V, E, _ptr(graph_ptr, "i32", **H), _ptr(child_ptr, "i32", **H), _ptr(child_idx, "i32", **H),
            _ptr(params, "f32", **H), int(x.shape[0]), _ptr(x, "f32", **H), _ptr(x_row, "i32", **H),
            _ptr(dh_out, "f32", **H), _ptr(dparams, "f32", **H), _ptr(dx, "f32", **H), _ptr(h_out, "f32", **H)))
        self.V, self.K = V, K

    def train_step_host_async(self, graph_ptr, child_ptr, child_idx, params, x, x_row, gamma, dparams,
                              gamma_rows=None):
        """cavs_train_step_host_async: pipelined step from pinned HOST arrays; `gamma` is dense [V, h] or,
        with `gamma_rows`, the cotangent rows of those vertices only.  Call sync() before reading dparams."""
        K = int(graph_ptr.shape[0]) - 1
        V = int(child_ptr.shape[0]) - 1
        E = int(child_idx.shape[0])
        H = dict(device=self.device, host_ok=True)
        n_g = int(gamma.shape[0]) if gamma is not None else 0
        self._keep_async = getattr(self, "_keep_async", [])[-3:] + [(graph_ptr, child_ptr, child_idx, params, x, x_row,
                                                                     gamma, gamma_rows, dparams)]
        self._check(_lib.cavs_train_step_host_async(
            self._ctx, K, V, E, _ptr(graph_ptr, "i32", **H), _ptr(child_ptr, "i32", **H), _ptr(child_idx, "i32", **H),
            _ptr(params, "f32", **H), int(x.shape[0]), _ptr(x, "f32", **H), _ptr(x_row, "i32", **H), n_g,
            _ptr(gamma_rows, "i32", **H), _ptr(gamma, "f32", **H), _ptr(dparams, "f32", **H)))
        self.V, self.K = V, K

    def close(self):
        if getattr(self, "_ctx", None):
            _lib.cavs_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
