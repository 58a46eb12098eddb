"""ctypes binding of libtpla.so (include/tpla.h).  Argument marshalling only.

Every function keeps the C name and raises ``TplaError`` on a non-OK status, with the
library's thread-local message.  Pointers are plain integers (``tensor.data_ptr()``) or
NumPy arrays for host buffers; streams are integers (``torch.cuda.current_stream().cuda_stream``).
There is no fallback: if the shared library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TPLA_LIB: an alternative build of the same library (kernel-variant experiments, tools/build_variant.py)
LIB_PATH = os.environ.get("TPLA_LIB") or os.path.join(_HERE, "libtpla.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2508_15881_b200.build` "
                      "(no CPU fallback exists for the TPLA hot path)")

if "TPLA_NCCL_LIB" not in os.environ:
    # the device API (f2(i)) must match the NCCL headers the library was compiled with (2.28): prefer
    # the NCCL that ships with torch over a system libnccl.so.2 found first on the loader path
    try:
        import nvidia.nccl  # type: ignore
        _nccl = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(_nccl):
            os.environ["TPLA_NCCL_LIB"] = _nccl
    except Exception:
        pass
_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

OK, ERR_INVALID_ARG, ERR_SHAPE, ERR_DIVISIBILITY, ERR_CAPACITY, ERR_CUDA, ERR_NCCL, ERR_UNSUPPORTED = range(8)
XFORM_IDENTITY, XFORM_HADAMARD, XFORM_PCA = 0, 1, 2
RMS_SLICED, RMS_EXACT, RMS_NONE = 0, 1, 2
DECODE_ACCUMULATE = 1
DECODE_STAGE_PRE, DECODE_STAGE_ATTN = 2, 4
ATTN_REUSE_PLAN = 1

_STATUS = {0: "OK", 1: "INVALID_ARG", 2: "SHAPE", 3: "DIVISIBILITY", 4: "CAPACITY", 5: "CUDA", 6: "NCCL",
           7: "UNSUPPORTED"}


class TplaError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn}: TPLA_{'ERR_' if status else ''}{_STATUS.get(status, status)}: {msg}")
        self.status = status


class tpla_config(C.Structure):
    _fields_ = [("h_q", C.c_int32), ("d_c", C.c_int32), ("d_r", C.c_int32), ("d_h", C.c_int32),
                ("D", C.c_int32), ("k", C.c_int32), ("g", C.c_int32), ("rank", C.c_int32),
                ("eps", C.c_float), ("sm_scale", C.c_float)]


class tpla_device_plan(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("rank", "shard", "head_block", "head_begin", "head_end", "lat_begin",
                                         "lat_end", "row_width", "h_loc", "w_lat")]


class tpla_weights(C.Structure):
    _fields_ = [("W_UK", C.c_void_p), ("W_UV", C.c_void_p), ("W_O", C.c_void_p), ("xform", C.c_void_p),
                ("xform_kind", C.c_int32), ("alpha_j", C.c_float), ("mu_j", C.c_float)]


class tpla_prefill_weights(C.Structure):
    _fields_ = [("W_UK", C.c_void_p), ("W_UV", C.c_void_p), ("W_O", C.c_void_p)]


class tpla_cache(C.Structure):
    _fields_ = [("base", C.c_void_p), ("block_table", C.c_void_p), ("num_pages", C.c_int64),
                ("page_size", C.c_int32), ("max_pages_per_seq", C.c_int32), ("row_stride", C.c_int32),
                ("batch", C.c_int32)]


_P = C.c_void_p
_I = C.c_int32
_S = C.c_size_t
_SIGS = {
    "tpla_version": ([], C.c_char_p),
    "tpla_last_error": ([], C.c_char_p),
    "tpla_launch_count": ([], C.c_int64),
    "tpla_make_plan": ([C.POINTER(tpla_config), C.POINTER(tpla_device_plan)], _I),
    "tpla_hadamard_signs": ([C.c_uint64, _I, _P], _I),
    "tpla_pca_alpha": ([_P, _I, _I, _P], _I),
    "tpla_weights_bytes": ([C.POINTER(tpla_config), _I, C.POINTER(_S), C.POINTER(_S), C.POINTER(_S), C.POINTER(_S)], _I),
    "tpla_convert_weights": ([C.POINTER(tpla_config), _I, C.c_uint64, _P, _P, _P, _P, _P, _P, _P,
                              C.POINTER(tpla_weights), _P], _I),
    "tpla_append_kv": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), C.POINTER(tpla_cache), _P, _P, _P, _P, _I,
                        _I, _P, _P], _I),
    "tpla_append_kv_norm_only": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), C.POINTER(tpla_cache), _P, _P, _P,
                                  _P, _I, _I, _P, _P, _P], _I),
    "tpla_prefill_mla": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), C.POINTER(tpla_cache), _P, _P, _P, _P,
                          _I, _P, _P], _I),
    "tpla_decode_workspace_bytes": ([C.POINTER(tpla_config), _I, _I, C.POINTER(_S)], _I),
    "tpla_decode": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), C.POINTER(tpla_cache), _P, _P, _P, _I, _I, _P,
                     _S, _P, _P, _I, _P, _P], _I),
    "tpla_decode_workspace_bytes_mtp": ([C.POINTER(tpla_config), _I, _I, _I, C.POINTER(_S)], _I),
    "tpla_prefill_workspace_bytes": ([C.POINTER(tpla_config), _I, _I, C.POINTER(_S)], _I),
    "tpla_prefill_attention": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), C.POINTER(tpla_cache), _P, _P, _I, _I,
                                _P, _S, _P, _P, _I, _P, _P], _I),
    "tpla_decode_v": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), C.POINTER(tpla_cache), _P, _P, _P, _I, _I, _I,
                       _P, _S, _P, _I, _I, _P], _I),
    "tpla_project_out": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), _P, _I, _I, _I, _P, _S, _P, _P, _I, _P,
                          _P, _P], _I),
    "tpla_project_out_sum": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), _P, _I, _I, _I, _I, _P, _S, _P, _P, _I,
                              _P, _P], _I),
    "tpla_decode_mtp": ([C.POINTER(tpla_config), C.POINTER(tpla_weights), C.POINTER(tpla_cache), _P, _P, _P, _I, _I,
                         _I, _P, _S, _P, _P, _I, _P, _P], _I),
    "tpla_decode_attention": ([C.POINTER(tpla_config), C.POINTER(tpla_cache), _P, _P, _P, _I, _I, _P, _S, _P, _P,
                               _P], _I),
    "tpla_decode_attention_ex": ([C.POINTER(tpla_config), C.POINTER(tpla_cache), _P, _P, _P, _I, _I, _P, _S, _P, _P,
                                  _I, _P], _I),
    "tpla_prefill_weights_bytes": ([C.POINTER(tpla_config), C.POINTER(_S), C.POINTER(_S), C.POINTER(_S)], _I),
    "tpla_convert_prefill_weights": ([C.POINTER(tpla_config), _P, _P, _P, _P, C.POINTER(tpla_prefill_weights), _P],
                                     _I),
    "tpla_prefill_mla_workspace_bytes": ([C.POINTER(tpla_config), _I, C.POINTER(_S)], _I),
    "tpla_prefill_mla_forward": ([C.POINTER(tpla_config), C.POINTER(tpla_prefill_weights), _P, _P, _P, _P, _I, _P, _S,
                                  _P, _P, _I, _P, _P], _I),
    "tpla_comm_unique_id": ([_P], _I),
    "tpla_comm_enable_fused_allreduce": ([_P, C.c_int64], _I),
    "tpla_decode_kernel_path": ([C.POINTER(tpla_config), _I], _I),
    "tpla_comm_fused_allreduce_mode": ([_P], _I),
    "tpla_comm_init": ([C.POINTER(_P), _P, _I, _I], _I),
    "tpla_comm_destroy": ([_P], _I),
    "tpla_sync": ([_P], _I),
    "tpla_profile_enable": ([_I], _I),
    "tpla_profile_collect": ([], _I),
    "tpla_profile_count": ([], _I),
    "tpla_profile_get": ([_I, C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)], _I),
    "tpla_profile_reset": ([], _I),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def _check(st: int, fn: str):
    if st != OK:
        raise TplaError(st, fn, _lib.tpla_last_error().decode())


def _ptr(x):
    """int | None | numpy array | torch tensor -> c_void_p"""
    if x is None:
        return None
    if isinstance(x, int):
        return C.c_void_p(x)
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("host array must be C-contiguous")
        return C.c_void_p(x.ctypes.data)
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(x.data_ptr())
    raise TypeError(type(x))


def tpla_version() -> str:
    return _lib.tpla_version().decode()


def tpla_last_error() -> str:
    return _lib.tpla_last_error().decode()


def tpla_launch_count() -> int:
    return int(_lib.tpla_launch_count())


def tpla_make_plan(cfg: tpla_config) -> tpla_device_plan:
    out = tpla_device_plan()
    _check(_lib.tpla_make_plan(C.byref(cfg), C.byref(out)), "tpla_make_plan")
    return out


def tpla_hadamard_signs(seed: int, d: int) -> np.ndarray:
    out = np.empty(d, np.float32)
    _check(_lib.tpla_hadamard_signs(C.c_uint64(seed & (2 ** 64 - 1)), d, _ptr(out)), "tpla_hadamard_signs")
    return out


def tpla_pca_alpha(lam: np.ndarray, g: int) -> np.ndarray:
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    out = np.empty(g, np.float32)
    _check(_lib.tpla_pca_alpha(_ptr(lam), lam.size, g, _ptr(out)), "tpla_pca_alpha")
    return out


def tpla_weights_bytes(cfg: tpla_config, xform_kind: int):
    a, b, c, d = _S(), _S(), _S(), _S()
    _check(_lib.tpla_weights_bytes(C.byref(cfg), xform_kind, C.byref(a), C.byref(b), C.byref(c), C.byref(d)),
           "tpla_weights_bytes")
    return a.value, b.value, c.value, d.value


def tpla_convert_weights(cfg, xform_kind, sign_seed, U_pca, alpha, mu, W_UK, W_UV, gamma, W_O, out: tpla_weights,
                         stream=0):
    alpha = np.ascontiguousarray(alpha, np.float32)
    mu = np.ascontiguousarray(mu, np.float32)
    U = None if U_pca is None else np.ascontiguousarray(U_pca, np.float32)
    arrs = [np.ascontiguousarray(x, np.uint16) for x in (W_UK, W_UV, gamma, W_O)]
    _check(_lib.tpla_convert_weights(C.byref(cfg), xform_kind, C.c_uint64(sign_seed & (2 ** 64 - 1)), _ptr(U),
                                     _ptr(alpha), _ptr(mu), *[_ptr(a) for a in arrs], C.byref(out), _ptr(stream)),
           "tpla_convert_weights")


def tpla_append_kv(cfg, w, cache, c_kv, k_pe, seq_idx, pos, n, rms_mode, n_dropped=None, stream=0):
    _check(_lib.tpla_append_kv(C.byref(cfg), C.byref(w), C.byref(cache), _ptr(c_kv), _ptr(k_pe), _ptr(seq_idx),
                               _ptr(pos), n, rms_mode, _ptr(n_dropped), _ptr(stream)), "tpla_append_kv")


def tpla_append_kv_norm_only(cfg, w, cache, c_kv, k_pe, seq_idx, pos, n, alpha, n_dropped=None, stream=0):
    a = np.ascontiguousarray(alpha, np.float32)
    _check(_lib.tpla_append_kv_norm_only(C.byref(cfg), C.byref(w), C.byref(cache), _ptr(c_kv), _ptr(k_pe),
                                         _ptr(seq_idx), _ptr(pos), n, a.size, _ptr(a), _ptr(n_dropped), _ptr(stream)),
           "tpla_append_kv_norm_only")


def tpla_prefill_mla(cfg, w, cache, c_kv, k_pe, seq_idx, pos, n, q=None, stream=0):
    _check(_lib.tpla_prefill_mla(C.byref(cfg), C.byref(w), C.byref(cache), _ptr(c_kv), _ptr(k_pe), _ptr(seq_idx),
                                 _ptr(pos), n, _ptr(q), _ptr(stream)), "tpla_prefill_mla")


def tpla_decode_workspace_bytes(cfg, B, max_seq_len) -> int:
    out = _S()
    _check(_lib.tpla_decode_workspace_bytes(C.byref(cfg), B, max_seq_len, C.byref(out)), "tpla_decode_workspace_bytes")
    return out.value


def tpla_decode(cfg, w, cache, q_nope, q_pe, seq_lens, B, max_seq_len, ws, ws_bytes, y, out=None, flags=0, comm=None,
                stream=0):
    _check(_lib.tpla_decode(C.byref(cfg), C.byref(w), C.byref(cache), _ptr(q_nope), _ptr(q_pe), _ptr(seq_lens), B,
                            max_seq_len, _ptr(ws), ws_bytes, _ptr(y), _ptr(out), flags, comm, _ptr(stream)),
           "tpla_decode")


def tpla_decode_workspace_bytes_mtp(cfg, B, n_q, max_seq_len) -> int:
    out = _S()
    _check(_lib.tpla_decode_workspace_bytes_mtp(C.byref(cfg), B, n_q, max_seq_len, C.byref(out)),
           "tpla_decode_workspace_bytes_mtp")
    return out.value


def tpla_decode_mtp(cfg, w, cache, q_nope, q_pe, seq_lens, B, n_q, max_seq_len, ws, ws_bytes, y, out=None, flags=0,
                    comm=None, stream=0):
    _check(_lib.tpla_decode_mtp(C.byref(cfg), C.byref(w), C.byref(cache), _ptr(q_nope), _ptr(q_pe), _ptr(seq_lens), B,
                                n_q, max_seq_len, _ptr(ws), ws_bytes, _ptr(y), _ptr(out), flags, comm, _ptr(stream)),
           "tpla_decode_mtp")


def tpla_prefill_workspace_bytes(cfg, L, max_pages_per_seq):
    n = _S(0)
    _check(_lib.tpla_prefill_workspace_bytes(C.byref(cfg), L, max_pages_per_seq, C.byref(n)),
           "tpla_prefill_workspace_bytes")
    return n.value


def tpla_prefill_attention(cfg, w, cache, q_nope, q_pe, seq, L, ws, ws_bytes, y, out=None, flags=0, comm=None,
                           stream=0):
    _check(_lib.tpla_prefill_attention(C.byref(cfg), C.byref(w), C.byref(cache), _ptr(q_nope), _ptr(q_pe), seq, L,
                                       _ptr(ws), ws_bytes, _ptr(y), _ptr(out), flags, comm, _ptr(stream)),
           "tpla_prefill_attention")


def tpla_decode_v(cfg, w, cache, q_nope, q_pe, seq_lens, B, n_q, max_seq_len, ws, ws_bytes, v_acc, n_chunks=1, flags=0,
                  stream=0):
    _check(_lib.tpla_decode_v(C.byref(cfg), C.byref(w), C.byref(cache), _ptr(q_nope), _ptr(q_pe), _ptr(seq_lens), B, n_q,
                              max_seq_len, _ptr(ws), ws_bytes, _ptr(v_acc), n_chunks, flags, _ptr(stream)),
           "tpla_decode_v")


def tpla_project_out(cfg, w, v_acc, R, n_chunks, chunk, ws, ws_bytes, y, out=None, flags=0, group_comm=None, comm=None,
                     stream=0):
    _check(_lib.tpla_project_out(C.byref(cfg), C.byref(w), _ptr(v_acc), R, n_chunks, chunk, _ptr(ws), ws_bytes, _ptr(y),
                                 _ptr(out), flags, group_comm, comm, _ptr(stream)), "tpla_project_out")


def tpla_project_out_sum(cfg, w, v_list, R, n_chunks, chunk, ws, ws_bytes, y, out=None, flags=0, comm=None, stream=0):
    """v_list: the co-located group's accumulators (tensors), summed in list order before W^O."""
    arr = (C.c_void_p * len(v_list))(*[_ptr(v) for v in v_list])
    _check(_lib.tpla_project_out_sum(C.byref(cfg), C.byref(w), C.cast(arr, C.c_void_p), len(v_list), R, n_chunks, chunk,
                                     _ptr(ws), ws_bytes, _ptr(y), _ptr(out), flags, comm, _ptr(stream)),
           "tpla_project_out_sum")


def tpla_prefill_weights_bytes(cfg: tpla_config):
    a, b, c = _S(), _S(), _S()
    _check(_lib.tpla_prefill_weights_bytes(C.byref(cfg), C.byref(a), C.byref(b), C.byref(c)),
           "tpla_prefill_weights_bytes")
    return a.value, b.value, c.value


def tpla_convert_prefill_weights(cfg, W_UK, W_UV, gamma, W_O, out: tpla_prefill_weights, stream=0):
    arrs = [np.ascontiguousarray(x, np.uint16) for x in (W_UK, W_UV, gamma, W_O)]
    _check(_lib.tpla_convert_prefill_weights(C.byref(cfg), *[_ptr(x) for x in arrs], C.byref(out), _ptr(stream)),
           "tpla_convert_prefill_weights")


def tpla_prefill_mla_workspace_bytes(cfg: tpla_config, L: int) -> int:
    n = _S()
    _check(_lib.tpla_prefill_mla_workspace_bytes(C.byref(cfg), L, C.byref(n)), "tpla_prefill_mla_workspace_bytes")
    return n.value


def tpla_prefill_mla_forward(cfg, w: tpla_prefill_weights, c_kv, k_pe, q_nope, q_pe, L, ws, ws_bytes, y, out=None,
                             flags=0, comm=None, stream=0):
    _check(_lib.tpla_prefill_mla_forward(C.byref(cfg), C.byref(w), _ptr(c_kv), _ptr(k_pe), _ptr(q_nope), _ptr(q_pe), L,
                                         _ptr(ws), ws_bytes, _ptr(y), _ptr(out), flags, comm, _ptr(stream)),
           "tpla_prefill_mla_forward")


def tpla_decode_attention(cfg, cache, q_lat, q_pe, seq_lens, B, max_seq_len, ws, ws_bytes, O, lse=None, stream=0):
    _check(_lib.tpla_decode_attention(C.byref(cfg), C.byref(cache), _ptr(q_lat), _ptr(q_pe), _ptr(seq_lens), B,
                                      max_seq_len, _ptr(ws), ws_bytes, _ptr(O), _ptr(lse), _ptr(stream)),
           "tpla_decode_attention")


def tpla_decode_attention_ex(cfg, cache, q_lat, q_pe, seq_lens, B, max_seq_len, ws, ws_bytes, O, lse=None, flags=0,
                             stream=0):
    _check(_lib.tpla_decode_attention_ex(C.byref(cfg), C.byref(cache), _ptr(q_lat), _ptr(q_pe), _ptr(seq_lens), B,
                                         max_seq_len, _ptr(ws), ws_bytes, _ptr(O), _ptr(lse), flags, _ptr(stream)),
           "tpla_decode_attention_ex")


def tpla_comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.tpla_comm_unique_id(C.cast(buf, C.c_void_p)), "tpla_comm_unique_id")
    return bytes(buf)


def tpla_comm_init(unique_id: bytes, world: int, rank: int):
    if len(unique_id) != 128:
        raise ValueError("unique id must be 128 bytes")
    buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
    out = C.c_void_p()
    _check(_lib.tpla_comm_init(C.byref(out), C.cast(buf, C.c_void_p), world, rank), "tpla_comm_init")
    return out


def tpla_comm_enable_fused_allreduce(comm, max_elems: int):
    """symmetric window + device communicator for the fused W^O epilogue + one-shot
    all-reduce (collective: every rank calls it)."""
    _check(_lib.tpla_comm_enable_fused_allreduce(comm, max_elems), "tpla_comm_enable_fused_allreduce")


def tpla_decode_kernel_path(cfg, B: int) -> int:
    """1: the tcgen05 K3, 0: the mma.sync K3 fallback; raises on an invalid shape."""
    r = int(_lib.tpla_decode_kernel_path(C.byref(cfg), B))
    if r < 0:
        raise TplaError(-r, "tpla_decode_kernel_path", _lib.tpla_last_error().decode())
    return r


def tpla_comm_fused_allreduce_mode(comm) -> int:
    """0: plain ncclAllReduce, 1: fused with peer loads (LSA), 2: fused through the NVLS multicast."""
    return int(_lib.tpla_comm_fused_allreduce_mode(comm))


def tpla_comm_destroy(comm):
    _check(_lib.tpla_comm_destroy(comm), "tpla_comm_destroy")


def tpla_sync(stream=0):
    _check(_lib.tpla_sync(_ptr(stream)), "tpla_sync")


def tpla_profile_enable(on: bool = True):
    _check(_lib.tpla_profile_enable(1 if on else 0), "tpla_profile_enable")


def tpla_profile_collect():
    _check(_lib.tpla_profile_collect(), "tpla_profile_collect")


def tpla_profile_count() -> int:
    return int(_lib.tpla_profile_count())


def tpla_profile_get(i: int):
    buf = C.create_string_buffer(64)
    ms = C.c_double()
    n = C.c_int64()
    _check(_lib.tpla_profile_get(i, buf, C.byref(ms), C.byref(n)), "tpla_profile_get")
    return buf.value.decode(), ms.value, n.value


def tpla_profile_reset():
    _check(_lib.tpla_profile_reset(), "tpla_profile_reset")


def profile_table() -> dict:
    """{kernel name: (total ms, launches)} accumulated since the last reset."""
    tpla_profile_collect()
    return {name: (ms, n) for name, ms, n in (tpla_profile_get(i) for i in range(tpla_profile_count()))}
