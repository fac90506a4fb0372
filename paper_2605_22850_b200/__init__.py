"""Python binding of libobjcache -- the B200-native ObjectCache hot path (arxiv 2605.22850).

Argument marshalling only: every step of the path (hashing, matching, descriptor resolution,
the layer-major gather + paged scatter kernels, layer-ready signalling, scheduling) runs inside
``libobjcache.so`` (C ABI in ``include/objcache.h``).  There is no Python or CPU fallback: if the
library is missing this import fails, and data-path calls on a machine without a GPU raise
``ObjcacheError(OC_ECUDA)``.

The boundary calls carry the names the paper's serving path uses (match -> descriptor
-> layer-ready waits): ``put_chunks``, ``match_prefix``, ``build_descriptor``,
``fetch_layerwise``, ``wait_layer``, ``schedule_bandwidth``.
"""
import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libobjcache.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2605_22850_b200/build.py` "
                      "(there is no fallback implementation)")
_lib = ctypes.CDLL(LIB_PATH)

# ---- constants (include/objcache.h) ------------------------------------------------------------
OC_OK, OC_EINVAL, OC_ENOMEM, OC_ENOTFOUND, OC_EIMMUTABLE = 0, -1, -2, -3, -4
OC_ERANGE, OC_EALIGN, OC_ECUDA, OC_EFULL, OC_ENOTSUP = -5, -6, -7, -8, -9
TIER_HBM, TIER_PINNED_HOST = 0, 1
DELIVER_LAYER_MAJOR, DELIVER_CHUNK_MAJOR = 0, 1
TARGET_PAGED, TARGET_FLAT = 0, 1
FETCH_PERSISTENT, FETCH_PER_LAYER = 0, 1
TENANT_WAITING, TENANT_RUNNING, TENANT_DONE, TENANT_CHUNKWISE = 0, 1, 2, 3
DISPATCH_INDEPENDENT, DISPATCH_WDRR = 0, 1
BATCH_BY_REQUEST, BATCH_BY_POSITION = 0, 1
COPY_LDST, COPY_BULK, COPY_CE, COPY_AUTO = 0, 1, 2, 3
FETCH_OVERLAP, FETCH_FIRST_LAYER_FULL, FETCH_YIELD, FETCH_LEAN = 1, 2, 4, 16
POLICIES = {"equal": 0, "kv_prop": 1, "bw_prop": 2, "stall_opt": 3, "cal_stall_opt": 4}

c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_u32p = ctypes.POINTER(ctypes.c_uint32)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i32p = ctypes.POINTER(ctypes.c_int32)


class CLayout(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_uint32), ("kv_heads", ctypes.c_uint32), ("head_dim", ctypes.c_uint32),
                ("elem_bytes", ctypes.c_uint32), ("chunk_tokens", ctypes.c_uint32)]


class CTarget(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("block_size", ctypes.c_uint32), ("first_token", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32), ("k_base", c_u64p), ("v_base", c_u64p),
                ("block_stride", ctypes.c_uint64), ("token_stride", ctypes.c_uint64),
                ("head_stride", ctypes.c_uint64), ("block_table", c_i32p), ("num_blocks", ctypes.c_uint64),
                ("flat_base", ctypes.c_uint64), ("flat_capacity", ctypes.c_uint64)]


class CFetchOpts(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_uint32), ("engine", ctypes.c_uint32), ("max_ctas", ctypes.c_uint32),
                ("unit_bytes", ctypes.c_uint32), ("pace_Bps", ctypes.c_double), ("pace_strict", ctypes.c_uint32),
                ("flags", ctypes.c_uint32)]


class CWdrrOpts(ctypes.Structure):
    _fields_ = [("weights", ctypes.POINTER(ctypes.c_double)), ("quantum_bytes", ctypes.c_uint64),
                ("entry_units", ctypes.c_uint32), ("hold_rates", ctypes.c_uint32),
                ("free_units", ctypes.POINTER(ctypes.c_uint64)), ("layer_packets", ctypes.c_uint32)]


class CProfile(ctypes.Structure):
    _fields_ = [("bytes_per_layer", ctypes.c_double), ("compute_per_layer_s", ctypes.c_double)]


_vp = ctypes.c_void_p
_SIGS = {
    "oc_geometry": [ctypes.POINTER(CLayout), c_u64p, c_u64p, c_u64p],
    "oc_select_mode": [ctypes.c_uint64, ctypes.c_uint64],
    "oc_sha256": [_vp, ctypes.c_uint64, c_u8p],
    "oc_chunk_keys": [c_u32p, ctypes.c_uint64, ctypes.c_uint32, _vp, _vp, ctypes.c_uint64, c_u64p],
    "oc_chunk_keys_batch": [_vp, _vp, _vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp, _vp, _vp],
    "oc_store_create": [ctypes.POINTER(CLayout), ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(_vp)],
    "oc_store_destroy": [_vp],
    "oc_store_count": [_vp, c_u64p],
    "oc_store_slab": [_vp, c_u64p, c_u64p],
    "oc_slot_pitch": [ctypes.POINTER(CLayout), ctypes.c_int, c_u64p],
    "oc_store_set_hot_layers": [_vp, ctypes.c_uint32],
    "oc_hot_layers_for": [ctypes.c_double, ctypes.c_double, ctypes.c_uint32, c_u32p],
    "oc_put_chunks": [_vp, _vp, _vp, ctypes.c_uint64, c_u64p, c_u64p],
    "oc_match_prefix": [_vp, c_u32p, ctypes.c_uint64, _vp, _vp, ctypes.c_uint64, c_u64p],
    "oc_store_lookup": [_vp, _vp, ctypes.c_uint64, c_u64p, c_u64p],
    "oc_store_attach_peer": [_vp, _vp],
    "oc_store_export": [_vp, _vp, c_u64p],
    "oc_store_import": [_vp, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(_vp)],
    "oc_build_descriptor": [_vp, _vp, ctypes.c_uint64, ctypes.POINTER(CLayout), ctypes.c_int,
                            ctypes.POINTER(CTarget), ctypes.POINTER(_vp), c_u64p],
    "oc_put_from_paged": [_vp, _vp, ctypes.c_uint64, ctypes.POINTER(CLayout), ctypes.POINTER(CTarget), _vp,
                          c_u64p, c_u64p],
    "oc_desc_free": [_vp],
    "oc_desc_info": [_vp, c_u64p, c_u64p, c_u64p],
    "oc_fetch_layerwise": [_vp, ctypes.POINTER(CFetchOpts), _vp],
    "oc_fetch_layers": [_vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(CFetchOpts), _vp],
    "oc_batch_create": [ctypes.POINTER(_vp), ctypes.c_uint32, ctypes.POINTER(_vp)],
    "oc_fetch_batch": [_vp, ctypes.POINTER(CFetchOpts), _vp],
    "oc_batch_free": [_vp],
    "oc_batch_set_order": [_vp, ctypes.c_int],
    "oc_scatter_flat": [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(CFetchOpts), _vp],
    "oc_fetch_batch_wdrr": [_vp, ctypes.POINTER(CFetchOpts), ctypes.POINTER(CWdrrOpts), _vp],
    "oc_wdrr_plan": [c_u64p, ctypes.c_uint32, c_u32p, ctypes.c_uint32, ctypes.POINTER(CWdrrOpts), c_u32p, c_u32p,
                     c_u32p, c_u32p, ctypes.c_uint64, c_u64p],
    "oc_wait_layer": [_vp, ctypes.c_uint32, _vp],
    "oc_sync_layer": [_vp, ctypes.c_uint32],
    "oc_layers_ready": [_vp, ctypes.POINTER(ctypes.c_uint32)],
    "oc_layer_times": [_vp, c_u64p],
    "oc_layer_times_async": [_vp, _vp, _vp],
    "oc_emulate_compute": [ctypes.c_uint64, _vp, _vp],
    "oc_trace_read": [c_u64p, ctypes.c_uint64],
    "oc_schedule_bandwidth": [ctypes.c_int, ctypes.POINTER(CProfile), ctypes.c_uint64, ctypes.c_double,
                              ctypes.c_double, ctypes.POINTER(ctypes.c_double)],
    "oc_pool_create": [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.POINTER(_vp)],
    "oc_pool_set_dispatch": [_vp, ctypes.c_int],
    "oc_pool_submit": [_vp, _vp, ctypes.c_double, _vp, c_u64p],
    "oc_pool_epoch": [_vp, c_u64p],
    "oc_pool_status": [_vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)],
    "oc_pool_destroy": [_vp],
    "oc_last_error": [],
    "oc_status_str": [ctypes.c_int],
    "oc_abi_version": [],
}
for _name, _args in _SIGS.items():
    try:
        _f = getattr(_lib, _name)
    except AttributeError as _e:
        raise ImportError(f"{LIB_PATH} is stale (no {_name}): rebuild with "
                          "`python paper_2605_22850_b200/build.py`") from _e
    _f.argtypes = _args
    _f.restype = ctypes.c_int
_lib.oc_last_error.restype = ctypes.c_char_p
_lib.oc_status_str.restype = ctypes.c_char_p

EXPORTED = tuple(_SIGS)


class ObjcacheError(RuntimeError):
    def __init__(self, code, message, bad_index=None):
        self.code = code
        self.bad_index = bad_index
        name = _lib.oc_status_str(code).decode()
        super().__init__(f"{name}: {message}" + (f" (index {bad_index})" if bad_index is not None else ""))


def _check(rc, bad_index=None):
    if rc != OC_OK:
        raise ObjcacheError(rc, _lib.oc_last_error().decode(errors="replace"),
                            bad_index if rc in (OC_ENOTFOUND, OC_EIMMUTABLE, OC_EFULL) else None)


# ---- helpers ------------------------------------------------------------------------------------
def _layout(lay) -> CLayout:
    if isinstance(lay, CLayout):
        return lay
    if hasattr(lay, "as_tuple"):
        lay = lay.as_tuple()
    elif hasattr(lay, "num_layers"):
        lay = (lay.num_layers, lay.kv_heads, lay.head_dim, lay.elem_bytes, lay.chunk_tokens)
    return CLayout(*[int(x) for x in lay])


def _stream(stream) -> Optional[int]:
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return int(stream.cuda_stream) or None
    return int(stream) or None


def _ptr(buf):
    """(address, nbytes, keepalive) of a contiguous numpy array, torch tensor or bytes."""
    if isinstance(buf, (bytes, bytearray)):
        arr = np.frombuffer(buf, dtype=np.uint8)
        return arr.ctypes.data, arr.nbytes, arr
    if isinstance(buf, np.ndarray):
        if not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return buf.ctypes.data, buf.nbytes, buf
    if hasattr(buf, "data_ptr"):  # torch.Tensor
        if not buf.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return int(buf.data_ptr()), buf.numel() * buf.element_size(), buf
    raise TypeError(f"unsupported buffer type {type(buf)}")


def _keys_array(keys) -> np.ndarray:
    if isinstance(keys, (list, tuple)) and keys and isinstance(keys[0], (bytes, bytearray)):
        keys = np.frombuffer(b"".join(keys), dtype=np.uint8)
    return np.ascontiguousarray(np.asarray(keys, dtype=np.uint8)).reshape(-1, 32)


def geometry(layout):
    """(row_bytes, S, chunk_bytes) of a layout (Eq. 1)."""
    row, S, ch = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    lay = _layout(layout)
    _check(_lib.oc_geometry(ctypes.byref(lay), ctypes.byref(row), ctypes.byref(S), ctypes.byref(ch)))
    return row.value, S.value, ch.value


def slot_pitch(layout, tier: int = 0) -> int:
    """oc_slot_pitch: byte distance between consecutive slots of a store slab of this layout/tier."""
    p = ctypes.c_uint64()
    lay = _layout(layout)
    _check(_lib.oc_slot_pitch(ctypes.byref(lay), int(tier), ctypes.byref(p)))
    return p.value


def select_mode(payload_W: int, theta: int) -> int:
    """Eq. 2 delivery mode (DELIVER_CHUNK_MAJOR if W < theta else DELIVER_LAYER_MAJOR)."""
    return _lib.oc_select_mode(int(payload_W), int(theta))


def sha256(data: bytes) -> bytes:
    out = (ctypes.c_uint8 * 32)()
    arr = np.frombuffer(bytes(data), dtype=np.uint8)
    _check(_lib.oc_sha256(arr.ctypes.data if arr.size else None, arr.size, out))
    return bytes(out)


def chunk_keys(tokens, chunk_tokens: int, parent: Optional[bytes] = None) -> np.ndarray:
    """[n, 32] uint8 keys of the complete chunk_tokens-blocks of ``tokens``."""
    t = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))
    n = t.size // int(chunk_tokens) if chunk_tokens else 0
    out = np.zeros((max(n, 1), 32), dtype=np.uint8)
    par = np.frombuffer(bytes(parent), dtype=np.uint8) if parent is not None else None
    cnt = ctypes.c_uint64()
    _check(_lib.oc_chunk_keys(t.ctypes.data_as(c_u32p), t.size, int(chunk_tokens),
                              par.ctypes.data if par is not None else None, out.ctypes.data, n, ctypes.byref(cnt)))
    return out[:cnt.value]


def chunk_keys_batch(token_streams, chunk_tokens: int, stream=None, parents=None):
    """Chain keys of many token streams in one GPU launch (oc_chunk_keys_batch): a list of uint32
    arrays in, a list of (floor(len/G), 32) uint8 arrays out.  `parents`: optional (R, 32) bytes."""
    import torch
    G = int(chunk_tokens)
    lens = [int(len(t)) for t in token_streams]
    nk = [n // G for n in lens] if G > 0 else [0] * len(lens)
    tok_off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64) if lens else np.zeros(0, np.uint64)
    key_off = np.concatenate([[0], np.cumsum(nk)[:-1]]).astype(np.uint64) if nk else np.zeros(0, np.uint64)
    flat = np.concatenate([np.asarray(t, dtype=np.uint32) for t in token_streams]) if lens else np.zeros(0, np.uint32)
    dev = torch.device("cuda", torch.cuda.current_device())
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64) if a.dtype == np.uint64 else
                                    np.ascontiguousarray(a).view(np.int32)).to(dev)
    t_tok, t_toff, t_len, t_koff = to(flat), to(tok_off), to(np.asarray(lens, np.uint64)), to(key_off)
    out = torch.empty((max(1, sum(nk)), 32), dtype=torch.uint8, device=dev)
    par = None
    if parents is not None:
        par = torch.from_numpy(np.ascontiguousarray(np.asarray(parents, dtype=np.uint8).reshape(-1, 32))).to(dev)
    s = torch.cuda.current_stream() if stream is None else stream
    _check(_lib.oc_chunk_keys_batch(t_tok.data_ptr(), t_toff.data_ptr(), t_len.data_ptr(), len(lens), G,
                                    par.data_ptr() if par is not None else None, out.data_ptr(), t_koff.data_ptr(),
                                    _stream(s)))
    s.synchronize()
    host = out.cpu().numpy()
    return [host[int(k0):int(k0) + n] for k0, n in zip(key_off, nk)]


def hot_layers_for(X_s: float, C_s: float, L: int) -> int:
    """Mirror depth (layers kept in HBM) that lets a host-tier fetch add no TTFT (Eq. 3)."""
    k = ctypes.c_uint32()
    _check(_lib.oc_hot_layers_for(float(X_s), float(C_s), int(L), ctypes.byref(k)))
    return k.value


def schedule_bandwidth(policy, s: Sequence[float], c: Sequence[float], cap_Bps: float,
                       delta_Bps: float = 0.0) -> np.ndarray:
    """Per-request rates in bytes/s (Sec. 3.6).  ``policy``: name in POLICIES or its code."""
    code = POLICIES[policy] if isinstance(policy, str) else int(policy)
    n = len(s)
    prof = (CProfile * max(n, 1))()
    for i in range(n):
        prof[i] = CProfile(float(s[i]), float(c[i]))
    out = (ctypes.c_double * max(n, 1))()
    _check(_lib.oc_schedule_bandwidth(code, prof, n, float(cap_Bps), float(delta_Bps), out))
    return np.array(out[:n], dtype=np.float64)


# ---- store ---------------------------------------------------------------------------------------
class Store:
    """Hash-addressed chunk store on one GPU (HBM slab or pinned, mapped host slab)."""

    def __init__(self, layout, capacity: int, tier: int = TIER_HBM, device: int = 0, _handle=None):
        self.layout = _layout(layout)
        self._peers = []
        if _handle is not None:
            self._h = _handle
        else:
            h = _vp()
            _check(_lib.oc_store_create(ctypes.byref(self.layout), int(tier), int(device), int(capacity),
                                        ctypes.byref(h)))
            self._h = h
        self.tier, self.device = tier, device

    def close(self, _destroy=_lib.oc_store_destroy):  # bound early: safe during interpreter exit
        if getattr(self, "_h", None):
            _destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def count(self) -> int:
        n = ctypes.c_uint64()
        _check(_lib.oc_store_count(self._h, ctypes.byref(n)))
        return n.value

    def set_hot_layers(self, hot_layers: int):
        """Pinned-host stores: mirror the first `hot_layers` layers of every chunk in HBM."""
        _check(_lib.oc_store_set_hot_layers(self._h, int(hot_layers)))

    @property
    def slab(self):
        b, n = ctypes.c_uint64(), ctypes.c_uint64()
        _check(_lib.oc_store_slab(self._h, ctypes.byref(b), ctypes.byref(n)))
        return b.value, n.value

    @property
    def slot_pitch(self) -> int:
        return slot_pitch(self.layout, self.tier)

    def put_chunks(self, keys, payloads) -> int:
        k = _keys_array(keys)
        addr, nbytes, keep = _ptr(payloads)
        if nbytes != k.shape[0] * geometry(self.layout)[2]:
            raise ValueError("payloads must hold n * L * S bytes")
        if getattr(payloads, "is_cuda", False):  # a torch producer may sit on a side stream
            import torch
            torch.cuda.current_stream(payloads.device).synchronize()
        n_new, bad = ctypes.c_uint64(), ctypes.c_uint64()
        rc = _lib.oc_put_chunks(self._h, k.ctypes.data, addr, k.shape[0], ctypes.byref(n_new), ctypes.byref(bad))
        del keep
        _check(rc, bad.value)
        return n_new.value

    def match_prefix(self, tokens, parent: Optional[bytes] = None) -> np.ndarray:
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))
        G = self.layout.chunk_tokens
        cap = t.size // G
        out = np.zeros((max(cap, 1), 32), dtype=np.uint8)
        par = np.frombuffer(bytes(parent), dtype=np.uint8) if parent is not None else None
        m = ctypes.c_uint64()
        _check(_lib.oc_match_prefix(self._h, t.ctypes.data_as(c_u32p), t.size,
                                    par.ctypes.data if par is not None else None, out.ctypes.data, cap,
                                    ctypes.byref(m)))
        return out[:m.value]

    def lookup(self, keys) -> np.ndarray:
        k = _keys_array(keys)
        out = np.zeros(max(k.shape[0], 1), dtype=np.uint64)
        bad = ctypes.c_uint64()
        _check(_lib.oc_store_lookup(self._h, k.ctypes.data, k.shape[0], out.ctypes.data_as(c_u64p),
                                    ctypes.byref(bad)), bad.value)
        return out[:k.shape[0]]

    def attach_peer(self, peer: "Store"):
        _check(_lib.oc_store_attach_peer(self._h, peer._h))
        self._peers.append(peer)

    def export(self) -> bytes:
        n = ctypes.c_uint64()
        _check(_lib.oc_store_export(self._h, None, ctypes.byref(n)))
        buf = (ctypes.c_uint8 * n.value)()
        _check(_lib.oc_store_export(self._h, buf, ctypes.byref(n)))
        return bytes(buf[:n.value])

    @classmethod
    def import_(cls, blob: bytes, device: int = 0) -> "Store":
        arr = np.frombuffer(blob, dtype=np.uint8)
        h = _vp()
        _check(_lib.oc_store_import(arr.ctypes.data, arr.size, int(device), ctypes.byref(h)))
        lay = CLayout(*np.frombuffer(blob[8:28], dtype=np.uint32).tolist())
        return cls(lay, 0, device=device, _handle=h)


# ---- targets and descriptors ----------------------------------------------------------------------
@dataclass
class PagedTarget:
    """Paged KV cache: see oc_target in include/objcache.h.  Addresses are device addresses."""
    k_base: Sequence[int]
    v_base: Sequence[int]
    block_stride: int
    token_stride: int
    head_stride: int
    block_size: int
    block_table: Sequence[int]
    first_token: int = 0


@dataclass
class FlatTarget:
    """The paper's flat client buffer: layer l's payload at base + l*N*S."""
    base: int
    capacity: int


def _fetch_opts(mode, engine, max_ctas, unit_bytes, pace_Bps, pace_strict, overlap, first_layer_full, yield_sms,
                lean):
    flags = ((FETCH_OVERLAP if overlap else 0) | (FETCH_FIRST_LAYER_FULL if first_layer_full else 0) |
             (FETCH_YIELD if yield_sms else 0) | (FETCH_LEAN if lean else 0))
    return CFetchOpts(int(mode), int(engine), int(max_ctas), int(unit_bytes), float(pace_Bps),
                      1 if pace_strict else 0, flags)


class Descriptor:
    def __init__(self, handle, store, layout, keepalive):
        self._h = handle
        self.store = store
        self.layout = layout
        self._keep = keepalive
        self.num_layers = layout.num_layers

    def close(self, _free=_lib.oc_desc_free):  # bound early: safe during interpreter exit
        if getattr(self, "_h", None):
            _free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def info(self):
        n, W, u = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(_lib.oc_desc_info(self._h, ctypes.byref(n), ctypes.byref(W), ctypes.byref(u)))
        return {"n_chunks": n.value, "payload_W": W.value, "units_per_layer": u.value}

    def fetch_layerwise(self, stream=None, mode=FETCH_PERSISTENT, engine=COPY_AUTO, max_ctas=0, unit_bytes=0,
                        pace_Bps=0.0, pace_strict=False, overlap=False, first_layer_full=False, yield_sms=False,
                        lean=False):
        """`overlap`: OC_FETCH_OVERLAP -- the launch may overlap the stream's previous fetch's tail
        (the caller guarantees that work does not touch this fetch's destination or sources).
        `first_layer_full`: OC_FETCH_FIRST_LAYER_FULL -- with max_ctas, layer 0 uses the whole GPU.
        `yield_sms`: OC_FETCH_YIELD -- layers after the first one unit per CTA (co-running prefill).
        `lean`: OC_FETCH_LEAN -- the smallest shared-memory ring per copy CTA."""
        o = _fetch_opts(mode, engine, max_ctas, unit_bytes, pace_Bps, pace_strict, overlap, first_layer_full,
                        yield_sms, lean)
        _check(_lib.oc_fetch_layerwise(self._h, ctypes.byref(o), _stream(stream)))

    def fetch_layers(self, l0: int, l1: int, stream=None, engine=COPY_AUTO, max_ctas=0, unit_bytes=0, lean=False,
                     yield_sms=False):
        """oc_fetch_layers: layers [l0, l1) of the current fetch (l0 = 0 opens a new one).
        `yield_sms` (l0 > 0, TMA engine): one unit per CTA, as OC_FETCH_YIELD's later layers."""
        o = _fetch_opts(FETCH_PERSISTENT, engine, max_ctas, unit_bytes, 0.0, False, False, False, yield_sms, lean)
        _check(_lib.oc_fetch_layers(self._h, int(l0), int(l1), ctypes.byref(o), _stream(stream)))

    def scatter_flat(self, flat_base: int, flat_capacity: int, stream=None, max_ctas=0, unit_bytes=0):
        """Scatter a layer-major payload [L][N][S] at device address flat_base into this
        descriptor's target (the client half of the paper's unfused flow)."""
        o = CFetchOpts(FETCH_PERSISTENT, COPY_BULK, int(max_ctas), int(unit_bytes), 0.0, 0, 0)
        _check(_lib.oc_scatter_flat(self._h, int(flat_base), int(flat_capacity), ctypes.byref(o), _stream(stream)))

    def wait_layer(self, layer: int, stream=None):
        _check(_lib.oc_wait_layer(self._h, int(layer), _stream(stream)))

    def sync_layer(self, layer: int):
        _check(_lib.oc_sync_layer(self._h, int(layer)))

    def layers_ready(self) -> int:
        n = ctypes.c_uint32(0)
        _check(_lib.oc_layers_ready(self._h, ctypes.byref(n)))
        return n.value

    def layer_times(self) -> np.ndarray:
        out = np.zeros(self.num_layers + 1, dtype=np.uint64)
        _check(_lib.oc_layer_times(self._h, out.ctypes.data_as(c_u64p)))
        return out

    def layer_times_async(self, out, stream=None):
        """Enqueue on `stream` the copy of the stamps into `out` (pinned host or device tensor /
        address of L + 1 u64), after the fetch completes; read it after synchronising `stream`."""
        addr = int(out.data_ptr()) if hasattr(out, "data_ptr") else int(out)
        _check(_lib.oc_layer_times_async(self._h, addr, _stream(stream)))


def _ctarget(target, lay):
    """(CTarget, keepalive list) for a PagedTarget / FlatTarget."""
    t = CTarget()
    keep = []
    if isinstance(target, FlatTarget):
        t.kind = TARGET_FLAT
        t.flat_base = int(target.base)
        t.flat_capacity = int(target.capacity)
    elif isinstance(target, PagedTarget):
        kb = np.ascontiguousarray(np.asarray(target.k_base, dtype=np.uint64))
        vb = np.ascontiguousarray(np.asarray(target.v_base, dtype=np.uint64))
        bt = np.ascontiguousarray(np.asarray(target.block_table, dtype=np.int32))
        keep += [kb, vb, bt]
        t.kind = TARGET_PAGED
        t.block_size = int(target.block_size)
        t.first_token = int(target.first_token)
        t.k_base = kb.ctypes.data_as(c_u64p)
        t.v_base = vb.ctypes.data_as(c_u64p)
        t.block_stride, t.token_stride, t.head_stride = (int(target.block_stride), int(target.token_stride),
                                                         int(target.head_stride))
        t.block_table = bt.ctypes.data_as(c_i32p)
        t.num_blocks = bt.size
        if kb.size != lay.num_layers or vb.size != lay.num_layers:
            raise ValueError("need one K and one V base per layer")
    else:
        raise TypeError("target must be PagedTarget or FlatTarget")
    return t, keep


class PreparedTarget:
    """A target converted to its C form once (for callers that build many descriptors over the
    same cache blocks: argument marshalling is then per call only for the keys)."""

    def __init__(self, target, layout):
        self.layout = _layout(layout)
        self.ctarget, self._keep = _ctarget(target, self.layout)


def build_descriptor(store: Store, keys, layout, target, delivery: int = DELIVER_LAYER_MAJOR) -> Descriptor:
    k = _keys_array(keys)
    if isinstance(target, PreparedTarget):
        lay, t, keep = target.layout, target.ctarget, [target]
    else:
        lay = _layout(layout)
        t, keep = _ctarget(target, lay)
    keep.append(k)
    h, bad = _vp(), ctypes.c_uint64()
    rc = _lib.oc_build_descriptor(store._h, k.ctypes.data, k.shape[0], ctypes.byref(lay), int(delivery),
                                  ctypes.byref(t), ctypes.byref(h), ctypes.byref(bad))
    _check(rc, bad.value)
    return Descriptor(h, store, lay, store)


class Batch:
    """Several descriptors fetched by one launch (layer-major across the batch)."""

    def __init__(self, descs: Sequence[Descriptor], order: int = BATCH_BY_REQUEST):
        self.descs = list(descs)
        arr = (_vp * len(self.descs))(*[d._h for d in self.descs])
        h = _vp()
        _check(_lib.oc_batch_create(arr, len(self.descs), ctypes.byref(h)))
        self._h = h
        if order != BATCH_BY_REQUEST:
            _check(_lib.oc_batch_set_order(h, int(order)))

    def set_order(self, order: int):
        _check(_lib.oc_batch_set_order(self._h, int(order)))

    def fetch(self, stream=None, max_ctas=0, unit_bytes=0, wdrr_weights=None, quantum_bytes=0, entry_units=0,
              hold_rates=False, engine=COPY_AUTO, free_units=None, layer_packets=0):
        """One launch for the whole batch.  With `wdrr_weights` (one per member) the claim order is
        weighted deficit round robin (oc_fetch_batch_wdrr, Alg. A2 line 7); `hold_rates` paces
        member i at wdrr_weights[i] bytes/s (Alg. A2 line 6); `free_units` (default: the members'
        mirrored layers) are claimed first and unpaced (reading c25); `layer_packets` = L makes a
        DRR packet a whole layer payload (Alg. A2 line 7 as written) instead of one unit."""
        o = CFetchOpts(FETCH_PERSISTENT, int(engine), int(max_ctas), int(unit_bytes), 0.0)
        if wdrr_weights is None:
            _check(_lib.oc_fetch_batch(self._h, ctypes.byref(o), _stream(stream)))
            return
        keep, opts = _wdrr_opts(wdrr_weights, quantum_bytes, entry_units, hold_rates, free_units, layer_packets)
        if len(wdrr_weights) != len(self.descs):
            raise ValueError("one WDRR weight per batch member")
        _check(_lib.oc_fetch_batch_wdrr(self._h, ctypes.byref(o), ctypes.byref(opts), _stream(stream)))

    def close(self, _free=_lib.oc_batch_free):  # bound early: safe during interpreter exit
        if getattr(self, "_h", None):
            _free(self._h)
            self._h = None

    def __del__(self):
        self.close()


def _wdrr_opts(weights, quantum_bytes, entry_units, hold_rates, free_units=None, layer_packets=0):
    """(arrays the options point into -- keep them alive across the call, options)."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    opts = CWdrrOpts(w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(quantum_bytes), int(entry_units),
                     1 if hold_rates else 0)
    opts.layer_packets = int(layer_packets)
    keep = [w]
    if free_units is not None:
        fu = np.ascontiguousarray(np.asarray(free_units, dtype=np.uint64))
        if len(fu) != len(w):
            raise ValueError("one free-unit count per request")
        opts.free_units = fu.ctypes.data_as(c_u64p)
        keep.append(fu)
    return keep, opts


def wdrr_plan(n_units, tile_bytes, weights, quantum_bytes=0, entry_units=0, hold_rates=False, free_units=None,
              layer_packets=0):
    """The WDRR claim order the library builds (host only): arrays (request, first unit, count,
    release us) of the entries.  free_units[i]: request i's leading units that are not paced;
    layer_packets = L: packets are whole layer payloads (n_units[i] / L units each)."""
    nu = np.ascontiguousarray(np.asarray(n_units, dtype=np.uint64))
    tb = np.ascontiguousarray(np.asarray(tile_bytes, dtype=np.uint32))
    keep, opts = _wdrr_opts(weights, quantum_bytes, entry_units, hold_rates, free_units, layer_packets)
    if len(weights) != len(nu):
        raise ValueError("one weight per request")
    n = ctypes.c_uint64()
    args = (nu.ctypes.data_as(c_u64p), len(nu), tb.ctypes.data_as(c_u32p), len(tb), ctypes.byref(opts))
    rc = _lib.oc_wdrr_plan(*args, None, None, None, None, 0, ctypes.byref(n))  # size query
    if rc != OC_ERANGE or n.value == 0:
        _check(rc)
    out = [np.zeros(n.value, dtype=np.uint32) for _ in range(4)]
    _check(_lib.oc_wdrr_plan(*args, *[o.ctypes.data_as(c_u32p) for o in out], n.value, ctypes.byref(n)))
    return tuple(out)


def fetch_batch(descs: Sequence[Descriptor], stream=None, **opts) -> "Batch":
    """Create a batch of descriptors and fetch it once; returns the (reusable) batch."""
    b = Batch(descs)
    b.fetch(stream, **opts)
    return b


class TenantPool:
    """Epoch admission of concurrent layerwise requests under a shared cap (Sec. 3.6, Alg. A2)."""

    def __init__(self, policy, cap_Bps: float, delta_Bps: float = 0.0, theta_bytes: int = 0,
                 dispatch: int = DISPATCH_INDEPENDENT):
        code = POLICIES[policy] if isinstance(policy, str) else int(policy)
        h = _vp()
        _check(_lib.oc_pool_create(code, float(cap_Bps), float(delta_Bps), int(theta_bytes), ctypes.byref(h)))
        self._h = h
        if dispatch != DISPATCH_INDEPENDENT:
            _check(_lib.oc_pool_set_dispatch(h, int(dispatch)))
        self._descs = []

    def submit(self, desc: Descriptor, compute_per_layer_s: float, stream=None) -> int:
        t = ctypes.c_uint64()
        _check(_lib.oc_pool_submit(self._h, desc._h, float(compute_per_layer_s), _stream(stream), ctypes.byref(t)))
        self._descs.append(desc)
        return t.value

    def epoch(self) -> int:
        n = ctypes.c_uint64()
        _check(_lib.oc_pool_epoch(self._h, ctypes.byref(n)))
        return n.value

    def status(self, ticket: int):
        st, r = ctypes.c_int(), ctypes.c_double()
        _check(_lib.oc_pool_status(self._h, int(ticket), ctypes.byref(st), ctypes.byref(r)))
        return st.value, r.value

    def close(self, _free=_lib.oc_pool_destroy):
        if getattr(self, "_h", None):
            _free(self._h)
            self._h = None

    def __del__(self):
        self.close()


# ---- the boundary calls, by the names the method uses ---------------------------------------------
def put_chunks(store: Store, keys, payloads) -> int:
    return store.put_chunks(keys, payloads)


def put_from_paged(store: Store, keys, layout, target: "PagedTarget", stream=None) -> int:
    """Offload: gather chunk j of a request from a paged cache into new store slots
    (asynchronous on `stream`); existing keys are deduplicated.  Returns the number of new keys."""
    k = _keys_array(keys)
    lay = _layout(layout)
    t, keep = _ctarget(target, lay)
    n_new, bad = ctypes.c_uint64(), ctypes.c_uint64()
    rc = _lib.oc_put_from_paged(store._h, k.ctypes.data, k.shape[0], ctypes.byref(lay), ctypes.byref(t),
                                _stream(stream), ctypes.byref(n_new), ctypes.byref(bad))
    del keep
    _check(rc, bad.value)
    return n_new.value


def match_prefix(store: Store, tokens, parent: Optional[bytes] = None) -> np.ndarray:
    return store.match_prefix(tokens, parent)


def fetch_layerwise(desc: Descriptor, stream=None, **opts):
    desc.fetch_layerwise(stream, **opts)


def fetch_layers(desc: Descriptor, l0: int, l1: int, stream=None, **opts):
    desc.fetch_layers(l0, l1, stream, **opts)


def wait_layer(desc: Descriptor, layer: int, stream=None):
    desc.wait_layer(layer, stream)


def emulate_compute(ns: int, stream=None, stamps=None):
    """Measurement support: a single-CTA %globaltimer spin of `ns` on `stream` standing in for a
    layer's compute window C_l; `stamps` (device tensor/address, 2 x u64) receives start and end."""
    addr = None if stamps is None else (int(stamps.data_ptr()) if hasattr(stamps, "data_ptr") else int(stamps))
    _check(_lib.oc_emulate_compute(int(ns), addr, _stream(stream)))


def trace_read() -> np.ndarray:
    """Measurement support: the last OC_TRACE=1 launch's ramp stamps, [2048 CTAs, 8] (ns, 0 = none)."""
    out = np.zeros(2048 * 8, dtype=np.uint64)
    _check(_lib.oc_trace_read(out.ctypes.data_as(c_u64p), out.size))
    return out.reshape(2048, 8)


def abi_version() -> int:
    return _lib.oc_abi_version()
