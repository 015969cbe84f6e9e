"""ctypes binding of libglad (include/glad.h).  Argument marshalling only:
every step of the decode path runs in the library's sm_100a kernels.  Torch is
used for device memory and streams.  There is no fallback: if libglad.so is
missing or fails to load, every call raises.
"""

import ctypes
import math
import os

import torch

# GLAD_LIB: debug/A-B override of the library file (default: the in-tree build)
_LIB_PATH = os.environ.get("GLAD_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libglad.so")
_lib = None

GLAD_OK, GLAD_ERR_INVALID_ARG, GLAD_ERR_UNSUPPORTED, GLAD_ERR_WORKSPACE, GLAD_ERR_CUDA = range(5)
MHA, MQA, GQA, GTA, GLA, MLA = range(6)


class GladError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"glad status {status}: {msg}")
        self.status = status


class CacheLayout(ctypes.Structure):
    """glad_cache_layout (include/glad.h)."""
    _fields_ = [("num_pages", ctypes.c_int32), ("page_size", ctypes.c_int32),
                ("n_heads_kv", ctypes.c_int32), ("d_head", ctypes.c_int32),
                ("d_rope", ctypes.c_int32), ("_reserved", ctypes.c_int32),
                ("row_stride", ctypes.c_int64)]

    @property
    def width(self):
        return self.n_heads_kv * self.d_head + self.d_rope

    def __repr__(self):
        return (f"CacheLayout(num_pages={self.num_pages}, page_size={self.page_size}, "
                f"n_heads_kv={self.n_heads_kv}, d_head={self.d_head}, d_rope={self.d_rope}, "
                f"row_stride={self.row_stride})")


def make_layout(num_pages, page_size, n_heads_kv, d_head, d_rope, row_stride=None):
    w = n_heads_kv * d_head + d_rope
    rs = row_stride if row_stride is not None else -(-w // 8) * 8
    return CacheLayout(int(num_pages), int(page_size), int(n_heads_kv), int(d_head), int(d_rope), 0, int(rs))


_I32P = ctypes.POINTER(ctypes.c_int32)
_VP = ctypes.c_void_p


def _sig(lib):
    L = ctypes.POINTER(CacheLayout)
    S = ctypes.c_int
    dec = [_VP, _VP, L, _VP, ctypes.c_int32, _VP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
           ctypes.c_float, ctypes.c_int32, _VP, _VP, _VP, ctypes.c_size_t, ctypes.c_int32, _VP]
    table = {
        "glad_last_error": ([], ctypes.c_char_p),
        "glad_version": ([], ctypes.c_char_p),
        "glad_debug_set_trace": ([_VP], None),
        "glad_debug_set_phase_mask": ([ctypes.c_int32], None),
        "glad_debug_set_tile": ([ctypes.c_int32], None),
        "glad_pool_bytes": ([L], ctypes.c_size_t),
        "glad_cache_append": ([L, _VP, _VP, ctypes.c_int32, _VP, _VP, ctypes.c_int32, ctypes.c_int32, _VP], S),
        "glad_paged_gather": ([L, _VP, _VP, ctypes.c_int32, _VP, ctypes.c_int32, ctypes.c_int32, _VP, _VP], S),
        "glad_decode_workspace_bytes": ([L] + [ctypes.c_int32] * 5, ctypes.c_size_t),
        "glad_gla_decode": (dec, S),
        "glad_mla_decode": (dec, S),
        "glad_gta_decode": (dec, S),
        "glad_splitkv_combine": ([_VP, _VP] + [ctypes.c_int32] * 5 + [_VP, _VP, _VP], S),
        "glad_tp_duplication": ([ctypes.c_int32] * 3, ctypes.c_int32),
        "glad_tp_shard": ([ctypes.c_int32] * 4 + [_I32P] * 4, S),
        "glad_seq_split_range": ([ctypes.c_int32] * 5 + [_I32P] * 2, S),
        "glad_gla_absorb_query": ([_VP, _VP, _VP, _VP] + [ctypes.c_int32] * 6 + [ctypes.c_float, _VP, _VP], S),
        "glad_cache_append_rope": ([L, _VP, _VP, ctypes.c_int32, _VP, _VP, _VP, ctypes.c_int32, ctypes.c_int32,
                                    ctypes.c_float, _VP], S),
        "glad_seq_split_rescale": ([_VP, ctypes.c_int32, ctypes.c_int32, _VP, ctypes.c_int64, ctypes.c_int32, _VP, _VP,
                                    _VP], S),
        "glad_kv_bytes_per_token_per_device": ([ctypes.c_int32] * 6, ctypes.c_int64),
        "glad_gla_prefill_workspace_bytes": ([ctypes.c_int32] * 6, ctypes.c_size_t),
        "glad_gla_prefill": ([_VP] * 7 + [ctypes.c_int32] * 7 + [ctypes.c_float, ctypes.c_float, _VP, _VP, _VP,
                                                                  ctypes.c_size_t, ctypes.c_int32, _VP], S),
    }
    for name, (args, res) in table.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


def lib():
    """Load libglad.so (raises if it is missing — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"libglad.so not built ({_LIB_PATH}); run __graft_entry__.build() "
                               "or `python -m paper_2505_21487_b200.build`")
        _lib = _sig(ctypes.CDLL(_LIB_PATH))
    return _lib


def exported_symbols():
    return ["glad_last_error", "glad_version", "glad_debug_set_trace", "glad_debug_set_phase_mask", "glad_debug_set_tile", "glad_pool_bytes", "glad_cache_append", "glad_paged_gather",
            "glad_decode_workspace_bytes", "glad_gla_decode", "glad_mla_decode",
            "glad_gta_decode", "glad_splitkv_combine", "glad_tp_duplication", "glad_tp_shard",
            "glad_seq_split_range", "glad_seq_split_rescale", "glad_gla_absorb_query", "glad_cache_append_rope",
            "glad_kv_bytes_per_token_per_device", "glad_gla_prefill_workspace_bytes", "glad_gla_prefill"]


def _check(status):
    if status != GLAD_OK:
        raise GladError(status, lib().glad_last_error().decode())


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _need(t, dtype, name, device=True):
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")


# ------------------------------------------------------------------ calls
def pool_bytes(layout):
    return lib().glad_pool_bytes(ctypes.byref(layout))


def cache_append(layout, pool, block_table, seqlens_before, rows, stream=None):
    """rows [B, n_new, width] bf16 -> pool (in place)."""
    _need(pool, torch.bfloat16, "pool"); _need(rows, torch.bfloat16, "rows")
    _need(block_table, torch.int32, "block_table"); _need(seqlens_before, torch.int32, "seqlens_before")
    B, n_new, w = rows.shape
    if w != layout.width:
        raise ValueError(f"rows width {w} != layout width {layout.width}")
    _check(lib().glad_cache_append(ctypes.byref(layout), _ptr(pool), _ptr(block_table), block_table.shape[1],
                                   _ptr(seqlens_before), _ptr(rows), B, n_new, _stream(stream)))


def paged_gather(layout, pool, block_table, seqlens, max_len, out=None, stream=None):
    _need(pool, torch.bfloat16, "pool"); _need(block_table, torch.int32, "block_table")
    _need(seqlens, torch.int32, "seqlens")
    B = seqlens.shape[0]
    if out is None:
        out = torch.empty(B, max_len, layout.width, dtype=torch.bfloat16, device=pool.device)
    _check(lib().glad_paged_gather(ctypes.byref(layout), _ptr(pool), _ptr(block_table), block_table.shape[1],
                                   _ptr(seqlens), B, max_len, _ptr(out), _stream(stream)))
    return out


def workspace_bytes(layout, B, Lq, H, variant=GLA, num_ctas=0):
    return lib().glad_decode_workspace_bytes(ctypes.byref(layout), B, Lq, H, variant, num_ctas)


class Workspace:
    """Reusable split-KV workspace (grows on demand; keeps CUDA-graph capture
    safe as long as it is sized before capture)."""

    def __init__(self, device="cuda"):
        self.buf = None
        self.device = device

    def get(self, nbytes):
        if nbytes == 0:
            return None
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        return self.buf


_default_ws = {}


def _decode(fn, variant, q, pool, layout, block_table, seqlens, softmax_scale, causal=True, out=None,
            lse=None, num_ctas=0, workspace=None, stream=None):
    _need(q, torch.bfloat16, "q"); _need(pool, torch.bfloat16, "pool")
    _need(block_table, torch.int32, "block_table"); _need(seqlens, torch.int32, "seqlens")
    B, Lq, H, _ = q.shape
    d_v = layout.d_head
    if out is None:
        out = torch.empty(B, Lq, H, d_v, dtype=torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty(B, Lq, H, dtype=torch.float32, device=q.device)
    nbytes = workspace_bytes(layout, B, Lq, H, variant, num_ctas)
    if workspace is None:
        # one default workspace per (device, stream): decodes in flight on
        # different streams never share plan / partial slots (concurrent
        # streams may also pass their own Workspace)
        key = (q.device, (stream or torch.cuda.current_stream(q.device)).cuda_stream)
        workspace = _default_ws.setdefault(key, Workspace(q.device))
    ws = workspace.get(nbytes)
    _check(fn(_ptr(q), _ptr(pool), ctypes.byref(layout), _ptr(block_table), block_table.shape[1], _ptr(seqlens),
              B, Lq, H, float(softmax_scale), 1 if causal else 0, _ptr(out), _ptr(lse), _ptr(ws), nbytes,
              num_ctas, _stream(stream)))
    return out, lse


def gla_decode(q, pool, layout, block_table, seqlens, softmax_scale, causal=True, **kw):
    """GLA decode (glad_gla_decode).  q [B, Lq, H, d_c + d_R] bf16."""
    return _decode(lib().glad_gla_decode, GLA, q, pool, layout, block_table, seqlens, softmax_scale, causal, **kw)


def mla_decode(q, pool, layout, block_table, seqlens, softmax_scale, causal=True, **kw):
    return _decode(lib().glad_mla_decode, MLA, q, pool, layout, block_table, seqlens, softmax_scale, causal, **kw)


def gta_decode(q, pool, layout, block_table, seqlens, softmax_scale, causal=True, **kw):
    return _decode(lib().glad_gta_decode, GTA, q, pool, layout, block_table, seqlens, softmax_scale, causal, **kw)


def splitkv_combine(o_part, lse_part, out=None, lse=None, stream=None):
    _need(o_part, torch.float32, "o_part"); _need(lse_part, torch.float32, "lse_part")
    S, B, Lq, H, d_v = o_part.shape
    if out is None:
        out = torch.empty(B, Lq, H, d_v, dtype=torch.bfloat16, device=o_part.device)
    if lse is None:
        lse = torch.empty(B, Lq, H, dtype=torch.float32, device=o_part.device)
    _check(lib().glad_splitkv_combine(_ptr(o_part), _ptr(lse_part), S, B, Lq, H, d_v, _ptr(out), _ptr(lse),
                                      _stream(stream)))
    return out, lse


def tp_duplication(N, g_q, h_q):
    return lib().glad_tp_duplication(N, g_q, h_q)


def tp_shard(h_q, n_kv_heads, N, rank):
    vals = [ctypes.c_int32() for _ in range(4)]
    _check(lib().glad_tp_shard(h_q, n_kv_heads, N, rank, *[ctypes.byref(v) for v in vals]))
    return tuple(v.value for v in vals)


def gla_absorb_query(q_nope, q_pe, w_uk, seqlens, rope_base=10000.0, out=None, stream=None):
    """q_nope [B,Lq,H,d_h], q_pe [B,Lq,H,d_R], w_uk [H,d_c,d_h] (bf16, device), seqlens [B] int32 ->
    q [B,Lq,H,d_c+d_R] bf16 for gla_decode / mla_decode (glad_gla_absorb_query)."""
    _need(q_nope, torch.bfloat16, "q_nope"); _need(q_pe, torch.bfloat16, "q_pe")
    _need(w_uk, torch.bfloat16, "w_uk"); _need(seqlens, torch.int32, "seqlens")
    if q_nope.dim() != 4 or q_pe.dim() != 4 or w_uk.dim() != 3:
        raise ValueError("q_nope / q_pe must be [B, Lq, H, d], w_uk [H, d_c, d_h]")
    B, Lq, H, d_h = q_nope.shape
    d_R = q_pe.shape[-1]
    d_c = w_uk.shape[1]
    if tuple(q_pe.shape[:3]) != (B, Lq, H):
        raise ValueError(f"q_pe shape {tuple(q_pe.shape)} does not match q_nope {tuple(q_nope.shape)}")
    if tuple(w_uk.shape) != (H, d_c, d_h):
        raise ValueError(f"w_uk shape {tuple(w_uk.shape)} != (H, d_c, d_h) = ({H}, {d_c}, {d_h})")
    if tuple(seqlens.shape) != (B,):
        raise ValueError(f"seqlens shape {tuple(seqlens.shape)} != ({B},)")
    if out is None:
        out = torch.empty((B, Lq, H, d_c + d_R), dtype=torch.bfloat16, device=q_nope.device)
    _need(out, torch.bfloat16, "out")
    if tuple(out.shape) != (B, Lq, H, d_c + d_R):
        raise ValueError(f"out shape {tuple(out.shape)} != {(B, Lq, H, d_c + d_R)}")
    _check(lib().glad_gla_absorb_query(_ptr(q_nope), _ptr(q_pe), _ptr(w_uk), _ptr(seqlens), B, Lq, H, d_h, d_c,
                                       d_R, float(rope_base), _ptr(out), _stream(stream)))
    return out


def cache_append_rope(layout, pool, block_table, seqlens_before, latent, k_pe, rope_base=10000.0, stream=None):
    """Append [latent || RoPE(k_pe, p)] rows (glad_cache_append_rope); latent [B,n,h*d], k_pe [B,n,d_R] bf16."""
    _need(pool, torch.bfloat16, "pool"); _need(block_table, torch.int32, "block_table")
    _need(seqlens_before, torch.int32, "seqlens_before")
    _need(latent, torch.bfloat16, "latent"); _need(k_pe, torch.bfloat16, "k_pe")
    if latent.dim() != 3 or k_pe.dim() != 3:
        raise ValueError("latent must be [B, n, n_heads_kv*d_head], k_pe [B, n, d_rope]")
    B, n = latent.shape[:2]
    if latent.shape[-1] != layout.n_heads_kv * layout.d_head:
        raise ValueError(f"latent width {latent.shape[-1]} != n_heads_kv*d_head = {layout.n_heads_kv * layout.d_head}")
    if tuple(k_pe.shape) != (B, n, layout.d_rope):
        raise ValueError(f"k_pe shape {tuple(k_pe.shape)} != {(B, n, layout.d_rope)}")
    if seqlens_before.numel() != B or block_table.dim() != 2 or block_table.shape[0] < B:
        raise ValueError("seqlens_before must be [B] and block_table [>= B, max_pages]")
    _check(lib().glad_cache_append_rope(ctypes.byref(layout), _ptr(pool), _ptr(block_table),
                                        block_table.shape[-1], _ptr(seqlens_before), _ptr(latent),
                                        _ptr(k_pe), B, n, float(rope_base), _stream(stream)))


def gla_prefill_workspace_bytes(B, Lmax, H, d_h, d_rope, num_ctas=0):
    return lib().glad_gla_prefill_workspace_bytes(B, Lmax, H, d_h, d_rope, num_ctas)


def gla_prefill(q_nope, q_pe, latent, k_pe, w_uk, w_uv, seqlens, softmax_scale, rope_base=10000.0, out=None,
                lse=None, num_ctas=0, workspace=None, stream=None):
    """Causal GLA prefill in the materialised form (glad_gla_prefill).  q_nope [B,L,H,d_h], q_pe [B,L,H,d_R],
    latent [B,L,h_c,d_c], k_pe [B,L,d_R] (unrotated), w_uk / w_uv [H,d_c,d_h] bf16, seqlens [B] int32 (device).
    Returns out [B,L,H,d_h] bf16 (head space), lse [B,L,H] fp32."""
    for t, n in ((q_nope, "q_nope"), (q_pe, "q_pe"), (latent, "latent"), (k_pe, "k_pe"), (w_uk, "w_uk"),
                 (w_uv, "w_uv")):
        _need(t, torch.bfloat16, n)
    _need(seqlens, torch.int32, "seqlens")
    B, L, H, d_h = q_nope.shape
    h_c, d_c = latent.shape[2], latent.shape[3]
    d_R = q_pe.shape[-1]
    if tuple(q_pe.shape[:3]) != (B, L, H) or tuple(latent.shape[:2]) != (B, L) or tuple(k_pe.shape) != (B, L, d_R):
        raise ValueError("q_pe / latent / k_pe shapes do not match q_nope")
    if tuple(w_uk.shape) != (H, d_c, d_h) or tuple(w_uv.shape) != (H, d_c, d_h):
        raise ValueError(f"w_uk / w_uv must be (H, d_c, d_h) = ({H}, {d_c}, {d_h})")
    if tuple(seqlens.shape) != (B,):
        raise ValueError("seqlens must be [B]")
    if out is None:
        out = torch.empty(B, L, H, d_h, dtype=torch.bfloat16, device=q_nope.device)
    if lse is None:
        lse = torch.empty(B, L, H, dtype=torch.float32, device=q_nope.device)
    nbytes = gla_prefill_workspace_bytes(B, L, H, d_h, d_R, num_ctas)
    if nbytes == 0:
        raise GladError(GLAD_ERR_UNSUPPORTED, "prefill: unsupported shape")
    if workspace is None:
        workspace = Workspace(q_nope.device)
    ws = workspace.get(nbytes)
    _check(lib().glad_gla_prefill(_ptr(q_nope), _ptr(q_pe), _ptr(latent), _ptr(k_pe), _ptr(w_uk), _ptr(w_uv),
                                  _ptr(seqlens), B, L, H, h_c, d_c, d_h, d_R, float(softmax_scale), float(rope_base),
                                  _ptr(out), _ptr(lse), _ptr(ws), nbytes, num_ctas, _stream(stream)))
    return out, lse


def seq_split_range(L, page_size, Lq, P, rank):
    """Token range [begin, end) of rank `rank` of a sequence-split group (glad_seq_split_range)."""
    b, e = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().glad_seq_split_range(int(L), int(page_size), int(Lq), int(P), int(rank), ctypes.byref(b),
                                      ctypes.byref(e)))
    return b.value, e.value


def seq_split_rescale(lse_all, rank, o, out=None, lse_out=None, stream=None):
    """lse_all [P, ...rows] fp32 (device), o [...rows, d_v] bf16 -> o * exp(lse_rank - lse) (fp32) and the
    merged lse (glad_seq_split_rescale)."""
    P = lse_all.shape[0]
    d_v = o.shape[-1]
    rows = o.numel() // d_v
    _need(lse_all, torch.float32, "lse_all"); _need(o, torch.bfloat16, "o")
    if lse_all[0].numel() != rows:
        raise ValueError(f"lse_all rows {lse_all[0].numel()} != o rows {rows}")
    out = torch.empty(o.shape, dtype=torch.float32, device=o.device) if out is None else out
    lse_out = torch.empty(lse_all.shape[1:], dtype=torch.float32, device=o.device) if lse_out is None else lse_out
    _check(lib().glad_seq_split_rescale(lse_all.data_ptr(), P, int(rank), o.data_ptr(), rows, d_v, out.data_ptr(),
                                        lse_out.data_ptr(), _stream(stream)))
    return out, lse_out


def kv_bytes_per_token_per_device(variant, n_kv_heads, d_head, d_rope, N, dtype_bytes=2):
    return lib().glad_kv_bytes_per_token_per_device(variant, n_kv_heads, d_head, d_rope, N, dtype_bytes)


TRACE_STRIDE = 8 + 12 * 128 + 32


def debug_set_trace(buf):
    """Debug timeline (see csrc/decode.cuh); buf: int64 CUDA tensor or None."""
    lib().glad_debug_set_trace(_ptr(buf) if buf is not None else ctypes.c_void_p(0))


def debug_set_phase_mask(mask):
    """Debug/benchmark: launch only plan (1) / decode (2) / merge (4)."""
    lib().glad_debug_set_phase_mask(int(mask))


def debug_set_tile(tokens):
    """Debug/benchmark: force 64-, 96- or 128-token KV tiles (0 = library choice)."""
    lib().glad_debug_set_tile(int(tokens))


def version():
    return lib().glad_version().decode()
