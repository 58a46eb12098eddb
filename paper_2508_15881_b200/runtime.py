"""Device-side state of one TPLA rank: converted weights, paged latent cache, workspace.

PyTorch is used only to allocate device memory and to name streams; every step of the
decode path runs inside libtpla.so (see ``_abi``).  This module is marshalling:
it sizes and allocates buffers, fills the C structs and calls the C entry points.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

from . import _abi as abi


@dataclasses.dataclass(frozen=True)
class LayerSpec:
    h_q: int
    d_c: int
    d_r: int
    d_h: int
    D: int
    eps: float = 1e-6
    sm_scale: float | None = None    # default 1/sqrt(d_h + d_r) (reading R1)

    @property
    def scale(self) -> float:
        return self.sm_scale if self.sm_scale is not None else 1.0 / math.sqrt(self.d_h + self.d_r)


def make_config(spec: LayerSpec, k: int, g: int, rank: int) -> abi.tpla_config:
    return abi.tpla_config(spec.h_q, spec.d_c, spec.d_r, spec.d_h, spec.D, k, g, rank, spec.eps, spec.scale)


def bf16_from_bits(bits: np.ndarray, device) -> torch.Tensor:
    """uint16 bf16 bit patterns (host) -> bf16 tensor on ``device`` (bitwise copy)."""
    t = torch.from_numpy(np.ascontiguousarray(bits, dtype=np.uint16).view(np.int16))
    return t.view(torch.bfloat16).to(device)


def bits_from_bf16(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


@dataclasses.dataclass(frozen=True)
class HeadBlockGroup:
    """One head block i as seen by one process.

    The g ranks {j·(k/g) + i} of head block i share W^O rows; the process holds `local_ranks`
    of them (they add into one v_acc), and `procs` are the processes holding any of them: v_acc
    is split into len(procs) column chunks, reduce-scattered over those processes, and this
    process projects chunk `chunk`."""
    head_block: int
    local_ranks: tuple
    procs: tuple
    chunk: int

    @property
    def n_chunks(self) -> int:
        return len(self.procs)


def head_block_groups(k: int, g: int, n_proc: int, proc: int) -> list[HeadBlockGroup]:
    """Head-block groups of process `proc` when k ranks (group-major plan: rank r has
    latent shard r div (k/g), head block r mod (k/g)) are spread over n_proc processes in
    contiguous runs of k/n_proc ranks (as bench.py assigns them)."""
    if k % n_proc or k % g:
        raise ValueError(f"k={k} over {n_proc} processes, g={g}")
    m, nb = k // n_proc, k // g
    out = []
    for i in range(nb):
        members = [j * nb + i for j in range(g)]
        procs = tuple(sorted({r // m for r in members}))
        local = tuple(r for r in members if r // m == proc)
        if local:
            out.append(HeadBlockGroup(i, local, procs, procs.index(proc)))
    return out


def group_process_sets(k: int, g: int, n_proc: int) -> list[tuple]:
    """Every distinct process set that must reduce-scatter (size > 1), in one global order (all
    processes create the communicators in this order, so overlapping sets cannot deadlock)."""
    sets = {grp.procs for p in range(n_proc) for grp in head_block_groups(k, g, n_proc, p)}
    return sorted(s for s in sets if len(s) > 1)


class TplaRank:
    """One device's share of a TPLA layer (plan, weights, cache, workspace)."""

    def __init__(self, spec: LayerSpec, *, k: int, g: int, rank: int, batch: int, max_seq_len: int,
                 page_size: int = 64, device="cuda", page_perm_seed: int | None = None, extra_pages: int = 0,
                 n_q: int = 1):
        self.spec = spec
        self.k, self.g, self.rank = k, g, rank
        self.cfg = make_config(spec, k, g, rank)
        self.plan = abi.tpla_make_plan(self.cfg)
        self.device = torch.device(device)
        self.batch = batch
        self.max_seq_len = max_seq_len
        self.page_size = page_size
        self.max_pages = (max_seq_len + page_size - 1) // page_size
        self.row_stride = ((self.plan.row_width + 63) // 64) * 64
        num_pages = batch * self.max_pages + extra_pages
        self.cache_buf = torch.zeros((num_pages, page_size, self.row_stride), dtype=torch.bfloat16, device=self.device)
        order = np.arange(num_pages, dtype=np.int64)
        if page_perm_seed is not None:      # scattered physical pages (exercises the page table)
            order = np.random.default_rng(page_perm_seed).permutation(num_pages)
        self.block_table_host = order[:batch * self.max_pages].reshape(batch, self.max_pages).astype(np.int32)
        self.block_table = torch.from_numpy(self.block_table_host).to(self.device)
        self.cache = abi.tpla_cache(self.cache_buf.data_ptr(), self.block_table.data_ptr(), num_pages, page_size,
                                    self.max_pages, self.row_stride, batch)
        self.n_q = n_q                  # query tokens per sequence the workspace is sized for (decode_mtp)
        self.ws_bytes = abi.tpla_decode_workspace_bytes_mtp(self.cfg, batch, n_q, max_seq_len)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.weights = None
        self._wbufs = None

    # ---- offline conversion
    def convert(self, W_UK, W_UV, gamma, W_O, *, xform: int, sign_seed: int = 0, U_pca=None, alpha=None, mu=None):
        """W_UK, W_UV [d_c, h_q d_h], gamma [d_c], W_O [h_q d_h, D]: host bf16 bits (uint16)."""
        g = self.g
        alpha = np.full(g, float(g)) if alpha is None else np.asarray(alpha, float)
        mu = alpha.copy() if mu is None else np.asarray(mu, float)
        nuk, nuv, nwo, nxf = abi.tpla_weights_bytes(self.cfg, xform)
        dev = self.device
        self._wbufs = (torch.empty(nuk // 2, dtype=torch.bfloat16, device=dev),
                       torch.empty(nuv // 2, dtype=torch.bfloat16, device=dev),
                       torch.empty(nwo // 2, dtype=torch.bfloat16, device=dev),
                       torch.empty(max(nxf // 4, 1), dtype=torch.float32, device=dev))
        w = abi.tpla_weights(self._wbufs[0].data_ptr(), self._wbufs[1].data_ptr(), self._wbufs[2].data_ptr(),
                             self._wbufs[3].data_ptr() if nxf else None, xform, 0.0, 0.0)
        abi.tpla_convert_weights(self.cfg, xform, sign_seed, U_pca, alpha, mu, W_UK, W_UV, gamma, W_O, w,
                                 stream_ptr())
        self.weights = w
        return w

    # ---- K1
    def append(self, c_kv: torch.Tensor, k_pe: torch.Tensor, seq_idx: torch.Tensor, pos: torch.Tensor,
               rms_mode: int = abi.RMS_SLICED, n_dropped: torch.Tensor | None = None, stream=None):
        n = int(c_kv.shape[0])
        abi.tpla_append_kv(self.cfg, self.weights, self.cache, c_kv, k_pe, seq_idx, pos, n, rms_mode, n_dropped,
                           stream_ptr(stream))

    def append_norm_only(self, c_kv, k_pe, seq_idx, pos, alpha, stream=None):
        """g = 1 rows normalised per slice (SURVEY f4 "norm only"): len(alpha) slices."""
        n = int(c_kv.shape[0])
        abi.tpla_append_kv_norm_only(self.cfg, self.weights, self.cache, c_kv, k_pe, seq_idx, pos, n, alpha,
                                     None, stream_ptr(stream))

    def prefill(self, c_kv, k_pe, seq_idx, pos, stream=None):
        n = int(c_kv.shape[0])
        abi.tpla_prefill_mla(self.cfg, self.weights, self.cache, c_kv, k_pe, seq_idx, pos, n, None,
                             stream_ptr(stream))

    # ---- prefill attention: the prompt's rows must be in the cache (prefill())
    def prefill_attention(self, q_nope, q_pe, seq: int, y, out=None, *, accumulate=False, comm=None, stream=None):
        """q_nope [L, h_q, d_h], q_pe [L, h_q, d_r]; y/out [L, D]: causal attention of the prompt held as
        cache sequence `seq` (positions 0..L-1), then W^UV, W^O (+ all-reduce)."""
        L = int(q_nope.shape[0])
        need = abi.tpla_prefill_workspace_bytes(self.cfg, L, self.max_pages)
        if getattr(self, "pf_ws", None) is None or self.pf_ws.numel() < need:
            self.pf_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        abi.tpla_prefill_attention(self.cfg, self.weights, self.cache, q_nope, q_pe, seq, L, self.pf_ws,
                                   self.pf_ws.numel(), y, out, abi.DECODE_ACCUMULATE if accumulate else 0, comm,
                                   stream_ptr(stream))

    # ---- K2..K5 (+ C1)
    def decode(self, q_nope, q_pe, seq_lens, y, out=None, *, B: int | None = None, accumulate=False, comm=None,
               stream=None):
        B = int(q_nope.shape[0]) if B is None else B
        abi.tpla_decode(self.cfg, self.weights, self.cache, q_nope, q_pe, seq_lens, B, self.max_seq_len, self.ws,
                        self.ws_bytes, y, out, abi.DECODE_ACCUMULATE if accumulate else 0, comm, stream_ptr(stream))

    def decode_mtp(self, q_nope, q_pe, seq_lens, y, out=None, *, accumulate=False, comm=None, stream=None):
        """Multi-token decode: q_nope [B, n_q, h_q, d_h], q_pe [B, n_q, h_q, d_r]; y/out [B * n_q, D]."""
        B, n_q = int(q_nope.shape[0]), int(q_nope.shape[1])
        abi.tpla_decode_mtp(self.cfg, self.weights, self.cache, q_nope, q_pe, seq_lens, B, n_q, self.max_seq_len,
                            self.ws, self.ws_bytes, y, out, abi.DECODE_ACCUMULATE if accumulate else 0, comm,
                            stream_ptr(stream))

    def decode_v(self, q_nope, q_pe, seq_lens, v_acc, *, n_chunks=1, accumulate=False, stage=None, stream=None):
        """K2..K5a into v_acc fp32 [n_chunks, B * n_q, H_loc * d_h / n_chunks] (f2(ii): the latent group
        sums v and shares one W^O read).  q_nope [B, h_q, d_h] or [B, n_q, h_q, d_h].
        stage: None (all), "pre" (K3p + K2 only) or "attn" (K3 + K45, after a "pre" call)."""
        B = int(q_nope.shape[0])
        n_q = int(q_nope.shape[1]) if q_nope.dim() == 4 else 1
        flags = (abi.DECODE_ACCUMULATE if accumulate else 0) | {None: 0, "pre": abi.DECODE_STAGE_PRE,
                                                                 "attn": abi.DECODE_STAGE_ATTN}[stage]
        abi.tpla_decode_v(self.cfg, self.weights, self.cache, q_nope, q_pe, seq_lens, B, n_q, self.max_seq_len, self.ws,
                          self.ws_bytes, v_acc, n_chunks, flags, stream_ptr(stream))

    def v_acc_shape(self, rows: int, n_chunks: int = 1):
        return (n_chunks, rows, self.plan.h_loc * self.spec.d_h // n_chunks)

    def project_out(self, v_acc, y, out=None, *, chunk=0, accumulate=False, group_comm=None, comm=None, stream=None):
        """[reduce-scatter v_acc over group_comm], y (+)= bf16(v_acc[chunk]) W^O[chunk's rows], [all-reduce]."""
        n_chunks, R = int(v_acc.shape[0]), int(v_acc.shape[1])
        abi.tpla_project_out(self.cfg, self.weights, v_acc, R, n_chunks, chunk, self.ws, self.ws_bytes, y, out,
                             abi.DECODE_ACCUMULATE if accumulate else 0, group_comm, comm, stream_ptr(stream))

    def project_out_sum(self, v_list, y, out=None, *, chunk=0, accumulate=False, comm=None, stream=None):
        """y (+)= bf16(Σ_i v_list[i][chunk]) W^O[chunk's rows] [, all-reduce]: a co-located group whose ranks
        wrote separate accumulators (decode_v without accumulate, e.g. on separate streams)."""
        n_chunks, R = int(v_list[0].shape[0]), int(v_list[0].shape[1])
        abi.tpla_project_out_sum(self.cfg, self.weights, list(v_list), R, n_chunks, chunk, self.ws, self.ws_bytes, y, out,
                                 abi.DECODE_ACCUMULATE if accumulate else 0, comm, stream_ptr(stream))

    def decode_attention(self, q_lat, q_pe, seq_lens, O, lse=None, *, B: int | None = None, reuse_plan=False,
                         stream=None):
        """reuse_plan: K3 without its schedule kernel, on the plan a previous call on this workspace left."""
        B = int(q_lat.shape[0]) if B is None else B
        abi.tpla_decode_attention_ex(self.cfg, self.cache, q_lat, q_pe, seq_lens, B, self.max_seq_len, self.ws,
                                     self.ws_bytes, O, lse, abi.ATTN_REUSE_PLAN if reuse_plan else 0, stream_ptr(stream))

    # ---- host view of the cache (tests)
    def cache_rows_bits(self, b: int, n: int) -> np.ndarray:
        """bf16 bits [n, row_stride] of sequence b's first n tokens, gathered through the page table."""
        t = torch.arange(n, device=self.cache_buf.device)
        pages = self.block_table[b].long()[t // self.page_size]
        return bits_from_bf16(self.cache_buf[pages, t % self.page_size])     # gathered on the device



class PrefillRank:
    """One device of the PD-separated MLA prefill: heads split over k devices,
    latent unsliced (g = 1), keys / values up-projected per head (tpla_prefill_mla_forward)."""

    def __init__(self, spec: LayerSpec, *, k: int, rank: int, max_len: int, device="cuda"):
        self.spec = spec
        self.k, self.rank = k, rank
        self.cfg = make_config(spec, k, 1, rank)
        self.device = torch.device(device)
        self.max_len = max_len
        self.ws_bytes = abi.tpla_prefill_mla_workspace_bytes(self.cfg, max_len)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.weights = None

    def convert(self, W_UK, W_UV, gamma, W_O):
        nuk, nuv, nwo = abi.tpla_prefill_weights_bytes(self.cfg)
        self._wbufs = tuple(torch.empty(n // 2, dtype=torch.bfloat16, device=self.device) for n in (nuk, nuv, nwo))
        w = abi.tpla_prefill_weights(*[b.data_ptr() for b in self._wbufs])
        abi.tpla_convert_prefill_weights(self.cfg, W_UK, W_UV, gamma, W_O, w, stream_ptr())
        self.weights = w
        return w

    def forward(self, c_kv, k_pe, q_nope, q_pe, y, out=None, *, accumulate=False, comm=None, stream=None):
        """c_kv [L, d_c] raw latents, k_pe [L, d_r], q_nope [L, h_q, d_h], q_pe [L, h_q, d_r] (bf16, device);
        y [L, D] fp32 (+= with accumulate), out [L, D] bf16 or None."""
        L = int(c_kv.shape[0])
        assert L <= self.max_len
        abi.tpla_prefill_mla_forward(self.cfg, self.weights, c_kv, k_pe, q_nope, q_pe, L, self.ws, self.ws_bytes, y, out,
                                     abi.DECODE_ACCUMULATE if accumulate else 0, comm, stream_ptr(stream))
