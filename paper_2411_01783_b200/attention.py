"""Device (B200) mirror of ``ringcp.attention`` — same names, arguments and errors.

Reference: /root/reference/pkg/src/ringcp/attention.py.  Blocks hold CUDA
tensors instead of frozen numpy arrays; every numeric operation runs in the
sm_100a kernels of ``_ringcp_b200.so`` (see include/ringcp_b200.h):

  gqa_attention      -> rcp_attn_fwd     (tcgen05/TMEM flash forward + LSE)
  merge_attention    -> rcp_merge_attn   (fp32 N-way LSE fold)
  metadata folding   -> rcp_fold_meta

Precision: Q/K/V are consumed as bf16 (fp32 inputs are rounded once), scores
and softmax sums accumulate in fp32, outputs and LSE are fp32.  The reference
uses fp64 everywhere; parity is within the north-star tolerance (|dO| <= 2e-2,
|dLSE| <= 1e-3 on bf16-exact inputs).  The structural guarantees are kept
exactly: LSE is the natural log, rows with no admitted key are 0 / -inf, padding
key rows are removed before any arithmetic (so padding is bitwise invisible),
and ``merge_attention([p]) is p``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = [
    "EmbeddingBlock",
    "GqaConfig",
    "PartialAttention",
    "admitted_pair_count",
    "gqa_attention",
    "merge_attention",
]

_INT32_MIN = -(2 ** 31)
KERNEL_HEAD_DIM = 128  # head_dim of the attention / decode kernels; smaller heads are zero-padded


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("ringcp_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _as_tensor(x, dtype=None, device=None) -> torch.Tensor:
    dev = device if device is not None else _device()
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=dtype) if dtype is not None else x.to(device=dev)
    else:
        arr = np.asarray(x)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        if dtype is not None:
            t = t.to(dtype)
    return t.contiguous()


@dataclass(frozen=True)
class GqaConfig:
    """Head geometry (attention.py:39-66): query head h reads kv head
    (h * n_kv_heads) // n_query_heads; scale defaults to 1/sqrt(head_dim)."""

    n_query_heads: int
    n_kv_heads: int
    head_dim: int
    scale: float | None = None

    def __post_init__(self):
        if self.n_query_heads < 1 or self.n_kv_heads < 1 or self.head_dim < 1:
            raise ValueError("head counts and head_dim must be positive")
        if self.n_query_heads % self.n_kv_heads != 0:
            raise ValueError(
                f"n_query_heads={self.n_query_heads} not divisible by n_kv_heads={self.n_kv_heads}")
        if self.scale is None:
            object.__setattr__(self, "scale", 1.0 / math.sqrt(self.head_dim))

    @property
    def query_to_kv_head(self) -> np.ndarray:
        return (np.arange(self.n_query_heads) * self.n_kv_heads) // self.n_query_heads


class EmbeddingBlock:
    """Token block on the GPU: ``data [T, H, D]``, int64 ``positions`` (-1 pad),
    bool ``valid``, int64 ``seq_ids`` (-1 pad) — attention.py:69-173.

    ``validate=True`` runs the reference's checks (finite valid rows,
    non-negative positions, strictly increasing positions per sequence,
    attention.py:85-106); it synchronises the device, so internal hot paths
    construct blocks with ``validate=False`` and a known ``n_valid``.
    Sequence ids of valid rows must fit in int32 (kernel metadata).
    Blocks are treated as immutable: no method writes into their tensors.
    """

    __slots__ = ("_data", "_positions", "_valid", "_seq_ids", "_n_valid", "_meta")

    def __init__(self, data, positions, valid, seq_ids, *, validate: bool = True,
                 n_valid: int | None = None, meta32=None):
        # Blocks built internally from prepared tensors (validate=False) stay on
        # their device; user-supplied data moves to the CUDA device.
        dev = data.device if (not validate and isinstance(data, torch.Tensor)) else None
        data = _as_tensor(data, device=dev)
        positions = _as_tensor(positions, torch.int64, dev)
        valid = _as_tensor(valid, torch.bool, dev)
        seq_ids = _as_tensor(seq_ids, torch.int64, dev)
        if data.dim() != 3:
            raise ValueError(f"data must be [tokens, heads, head_dim], got shape {tuple(data.shape)}")
        n = data.shape[0]
        if positions.shape != (n,) or valid.shape != (n,) or seq_ids.shape != (n,):
            raise ValueError("positions/valid/seq_ids must be 1-d arrays matching token count")
        self._data, self._positions, self._valid, self._seq_ids = data, positions, valid, seq_ids
        self._meta = {}
        if meta32 is not None:
            self._meta["q"] = meta32
        if validate:
            self._validate()
        elif n_valid is None:
            n_valid = int(valid.sum().item()) if n else 0
        if n_valid is not None:
            self._n_valid = int(n_valid)

    def _validate(self):
        n = self.n_tokens
        valid = self._valid
        if n and bool((valid & ~torch.isfinite(self._data).flatten(1).all(dim=1)).any()):
            raise ValueError("non-finite embedding data in valid rows")
        if n and bool((valid & (self._positions < 0)).any()):
            raise ValueError("valid tokens must have non-negative positions")
        self._n_valid = int(valid.sum().item()) if n else 0
        if self._n_valid:
            vs = self._seq_ids[valid]
            vp = self._positions[valid]
            if bool(((vs < _INT32_MIN + 2) | (vs > 2 ** 31 - 1)).any()):
                raise ValueError("sequence ids of valid tokens must fit in int32 (excluding the "
                                 "two padding sentinels)")
            if bool((vp > 2 ** 31 - 2).any()):
                raise ValueError("positions must be below 2**31 - 1")
            order = torch.sort(vs, stable=True).indices
            s2, p2 = vs[order], vp[order]
            bad = (s2[1:] == s2[:-1]) & (p2[1:] <= p2[:-1])
            if bool(bad.any()):
                sid = int(s2[1:][bad][0].item())
                raise ValueError(f"positions not strictly increasing within sequence {sid}")

    # -- reference fields
    @property
    def data(self) -> torch.Tensor:
        return self._data

    @property
    def positions(self) -> torch.Tensor:
        return self._positions

    @property
    def valid(self) -> torch.Tensor:
        return self._valid

    @property
    def seq_ids(self) -> torch.Tensor:
        return self._seq_ids

    @property
    def n_tokens(self) -> int:
        return int(self._data.shape[0])

    @property
    def n_heads(self) -> int:
        return int(self._data.shape[1])

    @property
    def head_dim(self) -> int:
        return int(self._data.shape[2])

    @property
    def n_valid(self) -> int:
        return self._n_valid

    # -- constructors (attention.py:108-138)
    @classmethod
    def from_tokens(cls, data, positions, seq_id: int = 0) -> "EmbeddingBlock":
        data = _as_tensor(data)
        n = data.shape[0]
        dev = data.device
        return cls(data, _as_tensor(positions, torch.int64), torch.ones(n, dtype=torch.bool, device=dev),
                   torch.full((n,), seq_id, dtype=torch.int64, device=dev))

    @classmethod
    def padding(cls, n_tokens: int, n_heads: int, head_dim: int, dtype=torch.float32) -> "EmbeddingBlock":
        if isinstance(dtype, type) or isinstance(dtype, np.dtype):
            dtype = torch.from_numpy(np.zeros(0, dtype=dtype)).dtype
        dev = _device()
        return cls(torch.zeros((n_tokens, n_heads, head_dim), dtype=dtype, device=dev),
                   torch.full((n_tokens,), -1, dtype=torch.int64, device=dev),
                   torch.zeros(n_tokens, dtype=torch.bool, device=dev),
                   torch.full((n_tokens,), -1, dtype=torch.int64, device=dev),
                   validate=False, n_valid=0)

    @staticmethod
    def concat(blocks: list["EmbeddingBlock"]) -> "EmbeddingBlock":
        if not blocks:
            raise ValueError("cannot concatenate zero blocks")
        return EmbeddingBlock(torch.cat([b.data for b in blocks], 0),
                              torch.cat([b.positions for b in blocks]),
                              torch.cat([b.valid for b in blocks]),
                              torch.cat([b.seq_ids for b in blocks]))

    def valid_only(self) -> "EmbeddingBlock":
        if self.n_valid == self.n_tokens:
            return self
        keep = self._valid
        return EmbeddingBlock(self._data[keep], self._positions[keep], self._valid[keep],
                              self._seq_ids[keep], validate=False, n_valid=self.n_valid)

    def pad_to(self, n_tokens: int) -> "EmbeddingBlock":
        if n_tokens < self.n_tokens:
            raise ValueError(f"cannot pad {self.n_tokens} tokens down to {n_tokens}")
        if n_tokens == self.n_tokens:
            return self
        pad = EmbeddingBlock.padding(n_tokens - self.n_tokens, self.n_heads, self.head_dim,
                                     dtype=self._data.dtype)
        out = EmbeddingBlock(torch.cat([self._data, pad.data]), torch.cat([self._positions, pad.positions]),
                             torch.cat([self._valid, pad.valid]), torch.cat([self._seq_ids, pad.seq_ids]),
                             validate=False, n_valid=self.n_valid)
        return out

    # -- device metadata
    def meta32(self, role: str):
        """(pos int32, seq int32) folded with the validity bit for role 'q' or 'k'
        (include/ringcp_b200.h); cached per block."""
        m = self._meta.get(role)
        if m is None:
            n = self.n_tokens
            dev = self._data.device
            pos = torch.empty(n, dtype=torch.int32, device=dev)
            seq = torch.empty(n, dtype=torch.int32, device=dev)
            lib = _lib.load()
            _lib.count("rcp_fold_meta")
            _lib.check(lib.rcp_fold_meta(_lib.ptr(self._positions), _lib.ptr(self._seq_ids),
                                         _lib.ptr(self._valid), n, 1 if role == "k" else 0,
                                         _lib.ptr(pos), _lib.ptr(seq), _lib.stream_handle()))
            m = (pos, seq)
            self._meta[role] = m
        return m

    def to_numpy(self):
        return (self._data.float().cpu().numpy(), self._positions.cpu().numpy(),
                self._valid.cpu().numpy(), self._seq_ids.cpu().numpy())

    def __repr__(self) -> str:
        return (f"EmbeddingBlock(tokens={self.n_tokens}, heads={self.n_heads}, "
                f"head_dim={self.head_dim}, dtype={self._data.dtype}, n_valid={self._n_valid})")


@dataclass(frozen=True)
class PartialAttention:
    """Output block plus per-(token, query head) natural-log LSE (attention.py:176-196)."""

    output: EmbeddingBlock
    lse: torch.Tensor

    def __post_init__(self):
        lse = _as_tensor(self.lse, torch.float32, self.output.data.device)
        if tuple(lse.shape) != (self.output.n_tokens, self.output.n_heads):
            raise ValueError(f"lse shape {tuple(lse.shape)} does not match output "
                             f"[{self.output.n_tokens}, {self.output.n_heads}]")
        object.__setattr__(self, "lse", lse)


def admitted_pair_count(q: EmbeddingBlock, k: EmbeddingBlock) -> int:
    """Number of admitted (query, key) pairs (attention.py:209-211), computed on
    device by sorted search instead of materialising the [Tq, Tk] mask."""
    if q.n_tokens == 0 or k.n_tokens == 0:
        return 0
    kv = k.valid
    kkey = (k.seq_ids[kv] << 32) + k.positions[kv]
    if kkey.numel() == 0:
        return 0
    kkey = torch.sort(kkey).values
    qv = q.valid
    qseq = q.seq_ids[qv]
    hi = torch.searchsorted(kkey, (qseq << 32) + q.positions[qv], right=True)
    lo = torch.searchsorted(kkey, qseq << 32, right=False)
    return int((hi - lo).sum().item())


def _check_kv_pair(k: EmbeddingBlock, v: EmbeddingBlock, cfg: GqaConfig):
    """attention.py:214-227."""
    if tuple(k.data.shape) != tuple(v.data.shape):
        raise ValueError(f"k/v shape mismatch: {tuple(k.data.shape)} vs {tuple(v.data.shape)}")
    same = (k.positions is v.positions and k.valid is v.valid and k.seq_ids is v.seq_ids)
    if not same and not (torch.equal(k.positions, v.positions) and torch.equal(k.valid, v.valid)
                         and torch.equal(k.seq_ids, v.seq_ids)):
        raise ValueError("k and v must carry identical positions/valid/seq_ids")
    if k.n_heads != cfg.n_kv_heads or k.head_dim != cfg.head_dim:
        raise ValueError(f"kv blocks are [{k.n_heads} x {k.head_dim}] but config wants "
                         f"[{cfg.n_kv_heads} x {cfg.head_dim}]")


def _bf16(t: torch.Tensor) -> torch.Tensor:
    return t if t.dtype == torch.bfloat16 else t.to(torch.bfloat16)


def attend_into(q_data: torch.Tensor, q_meta, k_data: torch.Tensor, v_data: torch.Tensor, k_meta,
                n_q_heads: int, n_kv_heads: int, scale: float, out: torch.Tensor, lse: torch.Tensor,
                mode: int, workspace: torch.Tensor | None = None, stream=None) -> None:
    """Raw kernel call: bf16 [T, H, 128] tensors (rows may be strided), folded
    int32 metadata, fp32 outputs written in place (mode overwrite / merge)."""
    lib = _lib.load()
    tq, tk = q_data.shape[0], k_data.shape[0]
    need = lib.rcp_attn_workspace_bytes(tq, tk)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 32), dtype=torch.uint8, device=q_data.device)
    _lib.count("rcp_attn_fwd")
    _lib.check(lib.rcp_attn_fwd(
        _lib.ptr(q_data), q_data.stride(0), _lib.ptr(k_data), k_data.stride(0),
        _lib.ptr(v_data), v_data.stride(0),
        _lib.ptr(q_meta[0]), _lib.ptr(q_meta[1]), _lib.ptr(k_meta[0]), _lib.ptr(k_meta[1]),
        tq, tk, n_q_heads, n_kv_heads, q_data.shape[2], float(scale),
        _lib.ptr(out), _lib.ptr(lse), mode, _lib.ptr(workspace), workspace.numel(),
        _lib.stream_handle(stream)))


def quantize_heads_e4m3(x: torch.Tensor, scale: torch.Tensor | None = None):
    """bf16 [T, H, 128] -> (e4m3 bytes [T, H, 128] uint8, per-head fp32 scales
    [H]): scales absmax / 448 rounded up to a power of two unless given
    (rcp_kv_calibrate_e4m3 / rcp_kv_quantize_e4m3)."""
    lib = _lib.load()
    x = _bf16(x)
    T, H, D = x.shape
    rows = x.reshape(T, H * D).contiguous()
    if scale is None:
        scale = torch.empty(H, dtype=torch.float32, device=x.device)
        ws = torch.empty(H, dtype=torch.int32, device=x.device)
        _lib.count("rcp_kv_calibrate_e4m3")
        _lib.check(lib.rcp_kv_calibrate_e4m3(_lib.ptr(rows), H * D, T, H, D, _lib.ptr(scale), _lib.ptr(ws),
                                             _lib.stream_handle()))
    out = torch.empty((T, H, D), dtype=torch.uint8, device=x.device)
    _lib.count("rcp_kv_quantize_e4m3")
    _lib.check(lib.rcp_kv_quantize_e4m3(_lib.ptr(out), H * D, 0, _lib.ptr(rows), H * D, T, H, D, _lib.ptr(scale),
                                        _lib.stream_handle()))
    return out, scale


def attend_into_qk8(q8: torch.Tensor, q_scale: torch.Tensor, q_meta, k8: torch.Tensor, k_scale: torch.Tensor,
                    v_data: torch.Tensor, k_meta, n_q_heads: int, n_kv_heads: int, scale: float,
                    out: torch.Tensor, lse: torch.Tensor, mode: int, workspace: torch.Tensor | None = None,
                    stream=None) -> None:
    """Raw call of the FP8-QK attention kernel (rcp_attn_fwd_qk8): e4m3 Q / K
    [T, H, 128] with per-head scales (value = scale * e4m3), bf16 V, folded
    int32 metadata, fp32 outputs written in place."""
    lib = _lib.load()
    tq, tk = q8.shape[0], k8.shape[0]
    need = lib.rcp_attn_workspace_bytes(tq, tk)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 32), dtype=torch.uint8, device=q8.device)
    _lib.count("rcp_attn_fwd")
    _lib.check(lib.rcp_attn_fwd_qk8(
        _lib.ptr(q8), q8.stride(0), _lib.ptr(k8), k8.stride(0), _lib.ptr(v_data), v_data.stride(0),
        _lib.ptr(q_meta[0]), _lib.ptr(q_meta[1]), _lib.ptr(k_meta[0]), _lib.ptr(k_meta[1]),
        tq, tk, n_q_heads, n_kv_heads, q8.shape[2], float(scale), _lib.ptr(q_scale), _lib.ptr(k_scale),
        _lib.ptr(out), _lib.ptr(lse), mode, _lib.ptr(workspace), workspace.numel(), _lib.stream_handle(stream)))


def gqa_attention_fp8(q: EmbeddingBlock, k: EmbeddingBlock, v: EmbeddingBlock, cfg: GqaConfig,
                      q_scale: torch.Tensor | None = None, k_scale: torch.Tensor | None = None) -> PartialAttention:
    """``gqa_attention`` with Q and K quantised to e4m3 (per head) and S = QK^T
    on the tensor cores' 8-bit path (an opt-in mode outside
    the bf16 parity contract: its result is that of ``gqa_attention`` on the
    dequantised Q / K).  head_dim must be 128."""
    if q.n_heads != cfg.n_query_heads or q.head_dim != cfg.head_dim:
        raise ValueError(f"query block is [{q.n_heads} x {q.head_dim}] but config wants "
                         f"[{cfg.n_query_heads} x {cfg.head_dim}]")
    _check_kv_pair(k, v, cfg)
    if cfg.head_dim != KERNEL_HEAD_DIM:
        raise ValueError(f"the e4m3 Q/K kernel takes head_dim == {KERNEL_HEAD_DIM}, got {cfg.head_dim}")
    if k.n_valid < k.n_tokens:
        k, v = k.valid_only(), v.valid_only()
    tq = q.n_tokens
    dev = q.data.device
    q8, qs = quantize_heads_e4m3(q.data, q_scale)
    k8, ks = quantize_heads_e4m3(k.data, k_scale)
    out = torch.empty((tq, cfg.n_query_heads, KERNEL_HEAD_DIM), dtype=torch.float32, device=dev)
    lse = torch.empty((tq, cfg.n_query_heads), dtype=torch.float32, device=dev)
    attend_into_qk8(q8, qs, q.meta32("q"), k8, ks, _bf16(v.data), k.meta32("k"), cfg.n_query_heads,
                    cfg.n_kv_heads, cfg.scale, out, lse, _lib.MODE_OVERWRITE)
    blk = EmbeddingBlock(out, q.positions, q.valid, q.seq_ids, validate=False, n_valid=q.n_valid)
    return PartialAttention(output=blk, lse=lse)


def gqa_attention(q: EmbeddingBlock, k: EmbeddingBlock, v: EmbeddingBlock, cfg: GqaConfig) -> PartialAttention:
    """Causal GQA attention of a query block against one key/value block
    (attention.py:230-282) on the tcgen05 kernel.  Key j is admitted for query i
    iff both are valid, same sequence, and positions[j] <= positions[i].
    head_dim <= 128 (smaller heads are zero-padded to the kernel's 128)."""
    if q.n_heads != cfg.n_query_heads or q.head_dim != cfg.head_dim:
        raise ValueError(f"query block is [{q.n_heads} x {q.head_dim}] but config wants "
                         f"[{cfg.n_query_heads} x {cfg.head_dim}]")
    _check_kv_pair(k, v, cfg)
    if cfg.head_dim > KERNEL_HEAD_DIM:
        raise ValueError(f"head_dim={cfg.head_dim} unsupported: the sm_100a kernels take head_dim <= "
                         f"{KERNEL_HEAD_DIM}")
    if k.n_valid < k.n_tokens:  # drop padding before any arithmetic (attention.py:253-255)
        k, v = k.valid_only(), v.valid_only()
    tq = q.n_tokens
    dev = q.data.device
    qd, kd, vd = _bf16(q.data), _bf16(k.data), _bf16(v.data)
    if cfg.head_dim < KERNEL_HEAD_DIM:
        # Smaller heads (e.g. the reference tests' D = 4 / 8) run on the same
        # kernel: zero columns change no Q.K dot product, the extra output
        # columns are V's zeros and are sliced off; the scale stays cfg.scale.
        pad = KERNEL_HEAD_DIM - cfg.head_dim
        qd, kd, vd = (torch.nn.functional.pad(x, (0, pad)).contiguous() for x in (qd, kd, vd))
    out = torch.empty((tq, cfg.n_query_heads, KERNEL_HEAD_DIM), dtype=torch.float32, device=dev)
    lse = torch.empty((tq, cfg.n_query_heads), dtype=torch.float32, device=dev)
    attend_into(qd, q.meta32("q"), kd, vd, k.meta32("k"),
                cfg.n_query_heads, cfg.n_kv_heads, cfg.scale, out, lse, _lib.MODE_OVERWRITE)
    if cfg.head_dim < KERNEL_HEAD_DIM:
        out = out[:, :, :cfg.head_dim].contiguous()
    blk = EmbeddingBlock(out, q.positions, q.valid, q.seq_ids, validate=False, n_valid=q.n_valid)
    return PartialAttention(output=blk, lse=lse)


def _check_same_query_geometry(a: PartialAttention, b: PartialAttention):
    """attention.py:285-296."""
    if tuple(a.output.data.shape) != tuple(b.output.data.shape):
        raise ValueError(f"partials are not query-shaped alike: {tuple(a.output.data.shape)} vs "
                         f"{tuple(b.output.data.shape)}")
    ao, bo = a.output, b.output
    same = ao.positions is bo.positions and ao.valid is bo.valid and ao.seq_ids is bo.seq_ids
    if not same and not (torch.equal(ao.positions, bo.positions) and torch.equal(ao.valid, bo.valid)
                         and torch.equal(ao.seq_ids, bo.seq_ids)):
        raise ValueError("partials disagree on query positions/valid/seq_ids")


def merge_rows_into(o_parts, lse_parts, out: torch.Tensor, lse_out: torch.Tensor, stream=None) -> None:
    """Raw fold of fp32 partials (list order) into out / lse_out."""
    lib = _lib.load()
    n = len(o_parts)
    rows = lse_out.numel()
    _lib.count("rcp_merge_attn")
    _lib.check(lib.rcp_merge_attn(_lib.ptr_array([_lib.ptr(t) for t in o_parts]),
                                  _lib.ptr_array([_lib.ptr(t) for t in lse_parts]), n, rows,
                                  out.shape[-1], _lib.ptr(out), _lib.ptr(lse_out),
                                  _lib.stream_handle(stream)))


def merge_attention(parts: list[PartialAttention]) -> PartialAttention:
    """Left fold of pairwise LSE merges in list order (attention.py:319-334);
    callers order parts by ascending source rank.  One part is returned as is."""
    if not parts:
        raise ValueError("cannot merge an empty list of partials")
    if len(parts) == 1:
        return parts[0]
    for p in parts[1:]:
        _check_same_query_geometry(parts[0], p)
    first = parts[0].output
    o_parts = [p.output.data.float().contiguous() for p in parts]
    l_parts = [p.lse.contiguous() for p in parts]
    out = torch.empty_like(o_parts[0])
    lse = torch.empty_like(l_parts[0])
    merge_rows_into(o_parts, l_parts, out, lse)
    blk = EmbeddingBlock(out, first.positions, first.valid, first.seq_ids, validate=False,
                         n_valid=first.n_valid)
    return PartialAttention(output=blk, lse=lse)
