"""ctypes binding of libsagips.so (include/sagips.h).  Argument marshalling
only: every step of the hot path runs in the library's CUDA kernels.  There
is no fallback -- importing this module fails loudly if the shared library
is missing or was built for another ABI."""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SAGIPS_LIB_VARIANT=x loads libsagips_x.so (same-box A/B builds, tests/tools/ab_lib.sh)
LIB_PATH = os.path.join(_HERE, "libsagips" + (("_" + os.environ["SAGIPS_LIB_VARIANT"])
                                              if os.environ.get("SAGIPS_LIB_VARIANT") else "") + ".so")

OK = 0
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "CONFIG", 3: "CUDA", 4: "NONFINITE", 5: "PROTOCOL",
          6: "STATE", 7: "TIMEOUT", 8: "UNSUPPORTED"}

MODE_NONE, MODE_ARAR, MODE_ARAR_ARAR, MODE_RMA_ARAR_ARAR, MODE_SYNC_ALLREDUCE, MODE_RMA_ALLGATHER, MODE_RMA_CHUNKED = range(7)
SAMPLER_QUADRATIC, SAMPLER_TABULATED = 0, 1
PREC_FP32, PREC_BF16 = 0, 1
DISC_AUTO, DISC_SIMT, DISC_TCGEN05 = 0, 1, 2
PRESET_DESK, PRESET_PAPER = 0, 1
STEP_LOCAL_ONLY, STEP_NO_ADAM_G, STEP_GRAPH = 1, 2, 4
IPC_HANDLE_BYTES = 64
NCCL_ID_BYTES = 128

(T_GEN_W, T_GEN_B, T_DISC_W, T_DISC_B, T_GEN_ADAM, T_DISC_ADAM, T_NOISE, T_RAW, T_C, T_EVENTS,
 T_REAL_IDX, T_HIST, T_LOGITS_D, T_LOGITS_G, T_DY, T_DRAW, T_GEN_DW, T_GEN_DB, T_DISC_DW,
 T_DISC_DB, T_REDUCED, T_STATS, T_REFERENCE, T_SHARD) = range(24)

_UINT32_TENSORS = {T_REAL_IDX, T_HIST}


class SagipsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"sagips: {STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [
        ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("group_size", ctypes.c_int32),
        ("outer_every", ctypes.c_int32), ("mode", ctypes.c_int32), ("staleness", ctypes.c_int32),
        ("reduce_mean", ctypes.c_int32), ("precision", ctypes.c_int32),
        ("noise_dim", ctypes.c_int32), ("gen_hidden", ctypes.c_int32), ("gen_depth", ctypes.c_int32),
        ("disc_hidden", ctypes.c_int32), ("disc_depth", ctypes.c_int32),
        ("param_samples", ctypes.c_int32), ("events_per_sample", ctypes.c_int32),
        ("reference_rows", ctypes.c_int64), ("shard_rows", ctypes.c_int64),
        ("gen_lr", ctypes.c_float), ("disc_lr", ctypes.c_float), ("leaky_slope", ctypes.c_float),
        ("adam_beta1", ctypes.c_float), ("adam_beta2", ctypes.c_float), ("adam_eps", ctypes.c_float),
        ("true_params", ctypes.c_float * 6),
        ("hist_bins", ctypes.c_int32), ("hist_lo", ctypes.c_float * 2), ("hist_hi", ctypes.c_float * 2),
        ("seed", ctypes.c_uint64),
        ("exchange_timeout_ms", ctypes.c_int32), ("phase_timing", ctypes.c_int32),
        ("disc_impl", ctypes.c_int32), ("sampler", ctypes.c_int32), ("sampler_grid", ctypes.c_int32),
        ("packet_biases", ctypes.c_int32), ("outer_rma", ctypes.c_int32), ("reserved", ctypes.c_int32 * 1),
    ]


class StepStats(ctypes.Structure):
    _fields_ = [("loss_d", ctypes.c_float), ("loss_g", ctypes.c_float), ("step", ctypes.c_uint64),
                ("outer_fired", ctypes.c_uint32), ("nonfinite", ctypes.c_uint32),
                ("wait_ns", ctypes.c_uint64), ("reserved", ctypes.c_uint64 * 4)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsagips.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    vp, sz, st = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    P = ctypes.POINTER
    sig = {
        "sagips_abi_version": ([], ctypes.c_int32),
        "sagips_config_init": ([P(Config), ctypes.c_int32], st),
        "sagips_workspace_size": ([P(Config), P(ctypes.c_size_t)], st),
        "sagips_create": ([P(Config), vp, sz, vp, P(vp)], st),
        "sagips_destroy": ([vp], st),
        "sagips_last_error": ([vp], ctypes.c_char_p),
        "sagips_sample_events": ([vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_uint32, ctypes.c_uint32, vp, vp, ctypes.c_int32, vp, vp, vp], st),
        "sagips_train_step": ([vp, ctypes.c_uint64, ctypes.c_uint32, vp], st),
        "sagips_train_step_host": ([vp, ctypes.c_uint64, ctypes.c_uint32, vp, vp, vp, vp], st),
        "sagips_push_generator_grad": ([vp, ctypes.c_uint64, vp], st),
        "sagips_pull_generator_grad": ([vp, ctypes.c_uint64, vp], st),
        "sagips_tensor_bytes": ([vp, ctypes.c_int32, P(ctypes.c_size_t)], st),
        "sagips_get": ([vp, ctypes.c_int32, vp, sz], st),
        "sagips_set": ([vp, ctypes.c_int32, vp, sz], st),
        "sagips_ipc_handle": ([vp, vp, sz], st),
        "sagips_connect_peers": ([vp, vp, sz], st),
        "sagips_window_ptr": ([vp, P(ctypes.c_uint64)], st),
        "sagips_connect_peers_local": ([vp, vp, sz], st),
        "sagips_nccl_unique_id": ([vp, sz], st),
        "sagips_connect_nccl": ([vp, vp, sz], st),
        "sagips_launch_count": ([vp, P(ctypes.c_uint64)], st),
        "sagips_graph_stats": ([vp, P(ctypes.c_uint64), P(ctypes.c_uint64)], st),
        "sagips_phase_times": ([vp, P(ctypes.c_float), ctypes.c_int32, P(ctypes.c_int32)], st),
        "sagips_kernel_times": ([vp, P(ctypes.c_float), ctypes.c_int32, P(ctypes.c_int32)], st),
        "sagips_timing_reset": ([vp], st),
        "sagips_debug_trace": ([vp, P(ctypes.c_size_t)], st),
        "sagips_predict_params": ([vp, vp, ctypes.c_int32, vp, vp], st),
        "sagips_sample_tabulated": ([vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, vp, vp], st),
        "sagips_sample_tabulated_bwd": ([vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, vp, vp, vp], st),
        "sagips_ensemble_stats": ([vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, vp, vp], st),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    if lib.sagips_abi_version() != 1:
        raise ImportError("libsagips.so ABI mismatch")
    return lib


lib = _load()
EXPORTED = [
    "sagips_abi_version", "sagips_config_init", "sagips_workspace_size", "sagips_create", "sagips_destroy",
    "sagips_last_error", "sagips_sample_events", "sagips_train_step", "sagips_push_generator_grad",
    "sagips_pull_generator_grad", "sagips_tensor_bytes", "sagips_get", "sagips_set", "sagips_ipc_handle",
    "sagips_connect_peers", "sagips_nccl_unique_id", "sagips_connect_nccl", "sagips_launch_count",
    "sagips_phase_times", "sagips_kernel_times", "sagips_timing_reset", "sagips_debug_trace",
    "sagips_predict_params", "sagips_ensemble_stats", "sagips_sample_tabulated", "sagips_sample_tabulated_bwd",
    "sagips_train_step_host", "sagips_window_ptr", "sagips_connect_peers_local", "sagips_graph_stats"]
NUM_PHASES = 7
PHASES = ["gen_fwd", "sampler", "disc_step", "gen_loss_through_disc", "sampler_bwd", "gen_bwd", "exchange_adam_g"]
NUM_KERNELS = 14
KERNELS = ["d_fwd_first", "d_fwd_mid", "d_fwd_head", "d_bwd_last", "d_bwd_mid", "d_bwd_first",
           "g_fwd_first", "g_fwd_mid", "g_fwd_head", "g_bwd_last", "g_bwd_mid", "g_bwd_dy", "g_fused", "d_fwd_fused"]


def _check(status, ctx=None):
    if status != OK:
        msg = lib.sagips_last_error(ctx).decode() if ctx else ""
        raise SagipsError(status, msg)


def config_init(preset=PRESET_DESK, **overrides):
    cfg = Config()
    _check(lib.sagips_config_init(ctypes.byref(cfg), preset))
    for k, v in overrides.items():
        if k in ("true_params", "hist_lo", "hist_hi"):
            arr = getattr(cfg, k)
            for i, x in enumerate(v):
                arr[i] = x
        else:
            setattr(cfg, k, v)
    return cfg


def workspace_size(cfg):
    n = ctypes.c_size_t()
    _check(lib.sagips_workspace_size(ctypes.byref(cfg), ctypes.byref(n)))
    return n.value


def nccl_unique_id():
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    _check(lib.sagips_nccl_unique_id(buf, NCCL_ID_BYTES))
    return buf.raw


def sample_events(c_ptr, k, m, seed, step, rank, stream_id, events_ptr, hist_ptr=None, bins=0,
                  lo=(0.0, 0.0), hi=(4.0, 4.0), stream=None):
    """Device pointers in, device pointers out (see sagips.h)."""
    lo_a = (ctypes.c_float * 2)(*lo)
    hi_a = (ctypes.c_float * 2)(*hi)
    _check(lib.sagips_sample_events(c_ptr, k, m, seed, step, rank, stream_id, events_ptr, hist_ptr, bins,
                                    ctypes.cast(lo_a, ctypes.c_void_p), ctypes.cast(hi_a, ctypes.c_void_p), stream))


def sample_tabulated(raw_ptr, k, m, G, seed, step, rank, stream_id, events_ptr, stream=None):
    """Tabulated-CDF sampler (R32): dev raw [k][6] -> dev events [k*m][2] (see sagips.h)."""
    _check(lib.sagips_sample_tabulated(raw_ptr, k, m, G, seed, step, rank, stream_id, events_ptr, stream))


def sample_tabulated_bwd(raw_ptr, k, m, G, seed, step, rank, stream_id, dy_ptr, draw_ptr, stream=None):
    """Its backward: dev dy [k*m][2] -> dev draw [k][6] (see sagips.h)."""
    _check(lib.sagips_sample_tabulated_bwd(raw_ptr, k, m, G, seed, step, rank, stream_id, dy_ptr, draw_ptr, stream))


def ensemble_stats(preds_ptr, M, k, P, p_true=None, stream=None):
    """Eq. 6-8 over dev preds [M][k][P] fp32 (see sagips.h): returns
    (p_hat, sigma, r_hat) as numpy float64 arrays of length P."""
    out = np.zeros(3 * P, dtype=np.float64)
    pt = None
    if p_true is not None:
        pt = np.ascontiguousarray(p_true, dtype=np.float64)
    _check(lib.sagips_ensemble_stats(preds_ptr, M, k, P, None if pt is None else pt.ctypes.data, out.ctypes.data,
                                     stream))
    return out[:P], out[P:2 * P], out[2 * P:]


class Context:
    """One rank.  `workspace_ptr` is a device allocation of at least
    workspace_size(cfg) bytes owned by the caller (e.g. a torch uint8 tensor
    kept alive in `self.keepalive`)."""

    def __init__(self, cfg, workspace_ptr, workspace_bytes, stream=None, keepalive=None):
        self.cfg = cfg
        self.keepalive = keepalive
        h = ctypes.c_void_p()
        st = lib.sagips_create(ctypes.byref(cfg), workspace_ptr, workspace_bytes, stream, ctypes.byref(h))
        if st != OK:
            raise SagipsError(st, "sagips_create failed")
        self.h = h

    def close(self):
        if self.h:
            lib.sagips_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def train_step(self, step, flags=0, stream=None):
        _check(lib.sagips_train_step(self.h, step, flags, stream), self.h)

    def predict_params(self, noise_ptr, k, c_out_ptr, stream=None):
        """Constrained parameters of the current generator for a dev noise
        batch [k][noise_dim] -> dev c_out [k][6] (sagips_predict_params)."""
        _check(lib.sagips_predict_params(self.h, noise_ptr, k, c_out_ptr, stream), self.h)

    def train_step_host(self, step, flags=0, noise_ptr=None, real_ptr=None, stats_ptr=None, stream=None):
        """train_step with the noise / real batch from host memory and the stats
        record copied back asynchronously (sagips_train_step_host)."""
        _check(lib.sagips_train_step_host(self.h, step, flags, noise_ptr, real_ptr, stats_ptr, stream), self.h)

    def push_generator_grad(self, step, stream=None):
        _check(lib.sagips_push_generator_grad(self.h, step, stream), self.h)

    def pull_generator_grad(self, step, stream=None):
        _check(lib.sagips_pull_generator_grad(self.h, step, stream), self.h)

    def tensor_bytes(self, which):
        n = ctypes.c_size_t()
        _check(lib.sagips_tensor_bytes(self.h, which, ctypes.byref(n)), self.h)
        return n.value

    def get(self, which):
        n = self.tensor_bytes(which)
        if which == T_STATS:
            s = StepStats()
            _check(lib.sagips_get(self.h, which, ctypes.byref(s), n), self.h)
            return s
        dt = np.uint32 if which in _UINT32_TENSORS else np.float32
        out = np.empty(n // 4, dtype=dt)
        _check(lib.sagips_get(self.h, which, out.ctypes.data, n), self.h)
        return out

    def set(self, which, arr):
        dt = np.uint32 if which in _UINT32_TENSORS else np.float32
        a = np.ascontiguousarray(arr, dtype=dt).reshape(-1)
        _check(lib.sagips_set(self.h, which, a.ctypes.data, a.nbytes), self.h)

    def ipc_handle(self):
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(lib.sagips_ipc_handle(self.h, buf, IPC_HANDLE_BYTES), self.h)
        return buf.raw

    def connect_peers(self, handles):
        blob = b"".join(handles)
        _check(lib.sagips_connect_peers(self.h, blob, len(blob)), self.h)

    def window_ptr(self):
        """Device address of this context's exchange window (0 if none)."""
        p = ctypes.c_uint64()
        _check(lib.sagips_window_ptr(self.h, ctypes.byref(p)), self.h)
        return p.value

    def connect_peers_local(self, ptrs):
        """Single-process wiring: the world's window addresses in rank order."""
        a = (ctypes.c_uint64 * len(ptrs))(*ptrs)
        _check(lib.sagips_connect_peers_local(self.h, a, len(ptrs)), self.h)

    def connect_nccl(self, uid):
        _check(lib.sagips_connect_nccl(self.h, uid, len(uid)), self.h)

    def phase_times(self):
        """Mean per-phase device milliseconds over the recent timed steps."""
        arr = (ctypes.c_float * NUM_PHASES)()
        n = ctypes.c_int32()
        _check(lib.sagips_phase_times(self.h, arr, NUM_PHASES, ctypes.byref(n)), self.h)
        return dict(zip(PHASES, list(arr))), n.value

    def kernel_times(self):
        """Mean device milliseconds per step of each tensor-core layer-pass class."""
        arr = (ctypes.c_float * NUM_KERNELS)()
        n = ctypes.c_int32()
        _check(lib.sagips_kernel_times(self.h, arr, NUM_KERNELS, ctypes.byref(n)), self.h)
        return dict(zip(KERNELS, list(arr))), n.value

    def timing_reset(self):
        _check(lib.sagips_timing_reset(self.h), self.h)

    def graph_stats(self):
        """(graph launches, graph instantiations) of SAGIPS_STEP_GRAPH steps."""
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib.sagips_graph_stats(self.h, ctypes.byref(a), ctypes.byref(b)), self.h)
        return a.value, b.value

    def launch_count(self):
        n = ctypes.c_uint64()
        _check(lib.sagips_launch_count(self.h, ctypes.byref(n)), self.h)
        return n.value


def debug_trace(with_ctas=False):
    """Timeline stamps of the tensor-core layer kernels (SAGIPS_TRACE=1):
    uint64 array [32 launches][4 CTAs][256 tiles][4]; with_ctas: also the
    per-CTA [32 launches][256 CTAs][12] records: (start, end) stamps in
    0, 1 and summed wait times (ns) per role in 4 + k (include/sagips.h)."""
    n = ctypes.c_size_t()
    _check(lib.sagips_debug_trace(None, ctypes.byref(n)))
    out = np.zeros(n.value // 8, dtype=np.uint64)
    _check(lib.sagips_debug_trace(out.ctypes.data, ctypes.byref(n)))
    k = 32 * 4 * 256 * 4
    tiles = out[:k].reshape(32, 4, 256, 4)
    return (tiles, out[k:].reshape(32, -1, 12)) if with_ctas else tiles
