"""ctypes binding of the C-ABI (include/tensched_b200.h).

The product path has no CPU fallback: if the sm_100a library is missing or
no B200 is visible, every scoring call raises.  Status codes map onto the
reference's exception hierarchy (pipeline_ir.py:20-37,
schedule_space.py:33).
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

import numpy as np

from .errors import IllegalActionError, PipelineError

LIB_PATH = pathlib.Path(os.environ.get(
    "TS_LIB", pathlib.Path(__file__).resolve().parent / "libtensched_b200.so"))

TS_OK = 0
TS_ERR_ILLEGAL = 4
TS_ERR_OVERFLOW = 5
MODE_EXACT = 0
MODE_FAST = 1

DECISION_DTYPE = np.dtype(
    [("split", "u1", 4), ("order", "u1", 8), ("n_loops", "u1"), ("vec", "u1"),
     ("flags", "u1"), ("anchor", "i1")]
)
assert DECISION_DTYPE.itemsize == 16


SPLIT_TABLE = np.array([0, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 32, 48, 64, 128, 255], dtype=np.uint8)
_SPLIT_CODE = np.full(256, 255, dtype=np.uint8)
_SPLIT_CODE[SPLIT_TABLE] = np.arange(16, dtype=np.uint8)
_VEC_CODE = np.full(256, 255, dtype=np.uint8)
_VEC_CODE[[1, 4, 8, 16]] = [0, 1, 2, 3]


def pack_records(recs: np.ndarray) -> np.ndarray | None:
    """16-byte ts_decision records -> the 8-byte wire format of
    ts_score_states_packed (None if a split factor or vector width falls
    outside the packed tables)."""
    sc = _SPLIT_CODE[recs["split"]]
    vc = _VEC_CODE[recs["vec"]]
    if np.any(sc == 255) or np.any(vc == 255):
        return None
    order = recs["order"].astype(np.uint64) & np.uint64(0xF)
    w = np.zeros(len(recs), dtype=np.uint64)
    for j in range(8):
        w |= order[:, j] << np.uint64(4 * j)
    w |= recs["n_loops"].astype(np.uint64) << np.uint64(32)
    for k in range(4):
        w |= sc[:, k].astype(np.uint64) << np.uint64(36 + 4 * k)
    w |= vc.astype(np.uint64) << np.uint64(52)
    w |= (recs["flags"].astype(np.uint64) & np.uint64(3)) << np.uint64(54)
    w |= (recs["anchor"].astype(np.int64) + 1).astype(np.uint64) << np.uint64(56)
    return w


class CudaUnavailableError(PipelineError):
    """The sm_100a extension or a B200 is not available (no CPU fallback)."""


_lib = None
_lib_lock = threading.Lock()


def _p(arr):
    # data_as: the pointer object keeps the array alive for the call, so a
    # temporary (`_p(x.copy())`) cannot be freed before the C side reads it
    return arr.ctypes.data_as(ctypes.c_void_p) if arr is not None else None


def load_library():
    """Load libtensched_b200.so (in-tree build) and declare signatures."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise CudaUnavailableError(
                f"{LIB_PATH.name} is not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(str(LIB_PATH))
        vp, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        sigs = {
            "ts_abi_version": ([], i32),
            "ts_last_error": ([vp], ctypes.c_char_p),
            "ts_ctx_create": ([i32, ctypes.POINTER(vp)], i32),
            "ts_ctx_destroy": ([vp], None),
            "ts_pipeline_upload": ([vp, vp, i64, ctypes.POINTER(i32)], i32),
            "ts_params_upload": ([vp, i32, vp, vp, vp, vp, f64, f64, vp, vp], i32),
            "ts_featurize_states": ([vp, i32, vp, vp, i64, i32, vp], i32),
            "ts_score_states": ([vp, i32, vp, vp, i64, i32, vp], i32),
            "ts_score_states_device": ([vp, i32, vp, vp, i64, i64, i32, vp], i32),
            "ts_score_states_packed": ([vp, i32, vp, vp, i64, i32, vp], i32),
            "ts_score_states_coded": ([vp, i32, vp, vp, i64, i32, vp], i32),
            "ts_decode_codes": ([vp, i32, vp, vp, i64, vp], i32),
            "ts_encode_codes_device": ([vp, i32, vp, vp, i64, vp], i32),
            "ts_encode_codes": ([vp, i32, vp, vp, i64, vp], i32),
            "ts_lstm_forward": ([vp, vp, i64, i64, i64, vp, vp, vp, vp, i64, f64, i32, vp], i32),
            "ts_lstm_backward": ([vp, vp, i64, i64, i64, vp, vp, vp, vp, i64, f64, vp, vp], i32),
            "ts_candidates": ([vp, i32, vp, i64, vp, i64, ctypes.POINTER(i64)], i32),
            "ts_check_action": ([vp, i32, vp, i64, vp], i32),
            "ts_greedy": ([vp, i32, f64, ctypes.POINTER(ctypes.c_uint64), vp,
                           ctypes.POINTER(i64), ctypes.POINTER(f64)], i32),
            "ts_greedy_stats": ([vp, ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
            "ts_beam": ([vp, i32, vp, i64, i32, vp, ctypes.POINTER(i64), ctypes.POINTER(f64)], i32),
            "ts_generate_states_device": ([vp, i32, ctypes.c_uint64, i64, vp, vp,
                                           ctypes.POINTER(i64)], i32),
            "ts_sync": ([vp], i32),
            "ts_stream": ([vp], vp),
            "ts_launch_count": ([vp], i64),
            "ts_set_timing": ([vp, i32], i32),
            "ts_kernel_times": ([vp, vp, vp, i32], i32),
            "ts_generate_schedules_device": ([vp, i32, ctypes.c_uint64, ctypes.c_uint64, i64, vp], i32),
            "ts_benchmark": ([vp, i32, vp, i64, vp, vp, vp, i64, vp], i32),
            "ts_featurize_rows_device": ([vp, i32, vp, vp, i64, vp], i32),
            "ts_init_rows": ([vp, i32, i32, vp], i32),
            "ts_train_load": ([vp, vp, i64, vp, i64, vp, vp, vp, vp, vp, i64, i32, i32], i32),
            "ts_train_set_params": ([vp, vp, i64], i32),
            "ts_train_get_params": ([vp, vp, i64], i32),
            "ts_train_grads": ([vp, vp, i64, i64, f64, vp, vp], i32),
            "ts_train_apply": ([vp, vp, f64, f64, vp], i32),
            "ts_train_forward": ([vp, vp, i64, vp], i32),
            "ts_train_set_mode": ([vp, i32], i32),
            "ts_score_children": ([vp, i32, vp, i64, vp, i64, f64, vp, vp, vp, vp], i32),
            "ts_score_states_coded_device": ([vp, i32, vp, vp, i64, i64, i32, vp], i32),
        }
        for name, (args, res) in sigs.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.ts_abi_version() != 1:
            raise CudaUnavailableError("ABI version mismatch")
        _lib = lib
        return lib


class Context:
    """One device context (stream, device buffers, uploaded pipelines/params)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = ctypes.c_void_p()
        rc = lib.ts_ctx_create(int(device), ctypes.byref(h))
        if rc != TS_OK:
            why = {7: "no sm_100 (B200) device visible", 6: "device log2 self-test failed",
                   2: "CUDA runtime failure"}.get(rc, f"status {rc}")
            raise CudaUnavailableError(f"cannot create a B200 context on device {device}: {why}")
        self.lib = lib
        self.h = h
        self.device = device
        self.lock = threading.RLock()
        self._pipelines = {}  # descriptor bytes -> id
        self._params_key = None

    def close(self):
        if self.h:
            self.lib.ts_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc == TS_OK:
            return
        msg = self.lib.ts_last_error(self.h).decode(errors="replace")
        if rc == TS_ERR_ILLEGAL:
            raise IllegalActionError(msg)
        raise PipelineError(f"tensched_b200 status {rc}: {msg}")

    # -- uploads -------------------------------------------------------------
    def pipeline_id(self, desc: np.ndarray) -> int:
        key = desc.tobytes()
        with self.lock:
            pid = self._pipelines.get(key)
            if pid is None:
                out = ctypes.c_int()
                self.check(self.lib.ts_pipeline_upload(self.h, _p(desc), desc.size,
                                                       ctypes.byref(out)))
                pid = self._pipelines[key] = out.value
            return pid

    def set_params(self, params):
        """Upload ValueModelParams (duck-typed, value_model.py:37-46) if changed."""
        arrs = [np.ascontiguousarray(a, dtype="<f8") for a in
                (params.Wx, params.Wh, params.b, params.w,
                 params.normalizer.mean, params.normalizer.std)]
        key = (int(params.hidden), float(params.b_out), float(params.target_scale),
               b"".join(a.tobytes() for a in arrs))
        with self.lock:
            if key == self._params_key:
                return
            self.check(self.lib.ts_params_upload(
                self.h, int(params.hidden), _p(arrs[0]), _p(arrs[1]), _p(arrs[2]),
                _p(arrs[3]), float(params.b_out), float(params.target_scale),
                _p(arrs[4]), _p(arrs[5])))
            self._params_key = key

    def launches(self) -> int:
        return int(self.lib.ts_launch_count(self.h))


_contexts: dict = {}


def host_context() -> Context:
    """Context for the library's host-side calls (candidate enumeration,
    legality).  Uses the device context when a B200 is present, otherwise a
    host-only context (device -1) that refuses every device entry point."""
    with _lib_lock:
        ctx = _contexts.get(-1)
    if ctx is not None:
        return ctx
    try:
        return context()
    except CudaUnavailableError:
        with _lib_lock:
            ctx = _contexts.get(-1)
        if ctx is None:
            ctx = Context(-1)
            with _lib_lock:
                _contexts[-1] = ctx
        return ctx


def context(device: int | None = None) -> Context:
    """Process-wide context per device (LOCAL_RANK by default)."""
    if device is None:
        device = int(os.environ.get("TS_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        try:
            import torch
            if torch.cuda.is_available() and os.environ.get("TS_DEVICE") is None:
                device = torch.cuda.current_device() if "LOCAL_RANK" not in os.environ else device
        except Exception:
            pass
    with _lib_lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lib_lock:
            _contexts[device] = ctx
    return ctx
