"""Device-resident decoder runtime: packed weights, the per-forward kernel
sequence, and CUDA-graph capture of draft / verify phases.

One forward over T query rows per sequence replaces T reference
``decode_step`` calls (/root/reference/pkg/src/quantspec/model.py:324-407):

  embed -> per layer [rmsnorm -> QKV linear (+RoPE, +k/v append into fp2)
  -> split-K attention over the store -> O linear (+residual) -> rmsnorm
  -> gate/up linear (+SiLU*up) -> down linear (+residual)] -> rmsnorm ->
  lm_head -> argmax

Every launch goes through the C ABI in libqsb200.so.  Kernel arguments that
change between steps (lengths, tokens) live in device memory, so a captured
graph stays valid across cycles; the only host sync per speculative cycle
is the readback of (accepted count, next token).
"""

from __future__ import annotations

import dataclasses

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError

SM_COUNT = 148
# queries per CTA in the quantised target view (<= 24: three 8-query tiles); QS_TGT_GROUP for A/B runs
_TGT_GROUP = int(__import__("os").environ.get("QS_TGT_GROUP", "24"))


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
# packed weights
# ---------------------------------------------------------------------------


@dataclass
class Geometry:
    num_layers: int
    hidden: int
    num_heads: int
    num_kv_heads: int
    head_dim: int
    mlp_hidden: int
    vocab: int
    max_positions: int
    rope_base: float = 10000.0
    norm_eps: float = 1e-5

    @property
    def nq(self) -> int:
        return self.num_heads * self.head_dim

    @property
    def nk(self) -> int:
        return self.num_kv_heads * self.head_dim


def rope_table(hd: int, base: float, max_pos: int):
    """cos/sin per (position, pair) computed exactly like Q/tensor.py:50-62 (f64 -> f32)."""
    torch = _torch()
    ex = np.arange(hd // 2, dtype=np.float64) * (2.0 / hd)
    inv = base ** -ex
    out = np.empty((max_pos, hd // 2, 2), dtype=np.float32)
    step = 1 << 14
    for p0 in range(0, max_pos, step):
        pos = np.arange(p0, min(max_pos, p0 + step), dtype=np.float64)[:, None]
        th = pos * inv[None, :]
        out[p0 : p0 + pos.shape[0], :, 0] = np.cos(th).astype(np.float32)
        out[p0 : p0 + pos.shape[0], :, 1] = np.sin(th).astype(np.float32)
    return torch.from_numpy(out).cuda()


def pack_f16(w):
    """[d_in, d_out] f32 CUDA tensor -> frag16 halves."""
    torch = _torch()
    d_in, d_out = (int(x) for x in w.shape)
    mt2 = (d_out // 16 + 1) // 2 * 2  # tile-pair-major frag16 layout pads to whole pairs
    out = torch.empty(mt2 * (d_in // 16) * 32 * 8, dtype=torch.float16, device=w.device)
    _lib.call("qs_pack_weights_f16", w.data_ptr(), d_in, d_out, out.data_ptr(), _lib.stream_ptr())
    return out


def interleave_cols(a, b):
    """[K, N] x 2 -> [K, 2N] with 16-column blocks alternating a, b (gate/up fusion:
    output tile 2j is gate tile j, 2j+1 is up tile j)."""
    K, N = (int(v) for v in a.shape)
    return _torch().stack([a.view(K, N // 16, 16), b.view(K, N // 16, 16)], dim=2).reshape(K, 2 * N).contiguous()


class PackedLinear:
    """One linear layer in device layout (frag16 or frag4 + params)."""

    def __init__(self, wmode: int, N: int, K: int, w, params=None, group: int = 0):
        self.wmode, self.N, self.K, self.w, self.params, self.group = wmode, N, K, w, params, group

    @classmethod
    def f16(cls, w):
        return cls(_lib.W_F16, int(w.shape[1]), int(w.shape[0]), pack_f16(w))

    @classmethod
    def f16_pair(cls, wa, wb):
        return cls.f16(interleave_cols(wa, wb))

    @classmethod
    def int4(cls, w, group: int):
        from .quant import quantize_weights_device

        _, _, _, frag, fp, g = quantize_weights_device(w, group, want_plane=False, want_frag=True)
        return cls(_lib.W_INT4, int(w.shape[1]), int(w.shape[0]), frag, fp, g)

    @classmethod
    def int4_pair(cls, wa, wb, group: int):
        return cls.int4(interleave_cols(wa, wb), group)

    def nbytes(self) -> int:
        b = self.w.numel() * self.w.element_size()
        if self.params is not None:
            b += self.params.numel() * self.params.element_size()
        return int(b)

    def algorithmic_bytes(self) -> float:
        """Bytes a GEMV must stream: 2 B/weight (f16) or 0.5 B/weight + 8 B/group (INT4)."""
        n_w = self.N * self.K
        if self.wmode == _lib.W_F16:
            return 2.0 * n_w
        return 0.5 * n_w + 8.0 * self.N * math.ceil(self.K / self.group)


class DeviceWeights:
    """Packed weights of one role (target fp16, or draft INT4) on the device."""

    def __init__(self, geo: Geometry, layers: list[dict], lm_head: PackedLinear, *, embedding, attn_norms,
                 mlp_norms, final_norm, rope, wmode: int):
        self.geo = geo
        self.layers = layers  # dict(qkv, o, gu, down)
        self.lm_head = lm_head
        self.embedding = embedding
        self.attn_norms = attn_norms
        self.mlp_norms = mlp_norms
        self.final_norm = final_norm
        self.rope = rope
        self.wmode = wmode

    def nbytes(self) -> int:
        return sum(pl.nbytes() for lw in self.layers for pl in lw.values()) + self.lm_head.nbytes()

    def algorithmic_bytes(self) -> float:
        return sum(pl.algorithmic_bytes() for lw in self.layers for pl in lw.values()) + self.lm_head.algorithmic_bytes()


def build_device_weights(geo: Geometry, layer_mats, embedding, final_norm, lm_head, attn_norms, mlp_norms, *,
                         int4_group: int | None = None, rope=None, want_fp16: bool = True,
                         head_shard: tuple[int, int] | None = None):
    """layer_mats: iterable yielding per-layer dicts of CUDA f32 [d_in, d_out] tensors.

    Returns (fp16 DeviceWeights or None, INT4 DeviceWeights or None); tensors
    are consumed one layer at a time so only packed copies stay resident.
    ``head_shard=(rank, world)`` keeps only this rank's query / key / value head
    columns of the QKV projection (KV-head sharding); the output
    projection, MLP and lm_head stay replicated.
    """
    torch = _torch()
    rope = rope if rope is not None else rope_table(geo.head_dim, geo.rope_base, geo.max_positions)
    f_layers, q_layers = [], []
    for mats in layer_mats:
        wq, wk, wv = mats["wq"], mats["wk"], mats["wv"]
        if head_shard is not None:
            r, n = head_shard
            qn, kn = geo.nq // n, geo.nk // n
            wq, wk, wv = wq[:, r * qn:(r + 1) * qn], wk[:, r * kn:(r + 1) * kn], wv[:, r * kn:(r + 1) * kn]
        qkv = torch.cat([wq, wk, wv], dim=1)
        if want_fp16:
            f_layers.append(dict(qkv=PackedLinear.f16(qkv), o=PackedLinear.f16(mats["wo"]),
                                 gu=PackedLinear.f16_pair(mats["w_gate"], mats["w_up"]),
                                 down=PackedLinear.f16(mats["w_down"])))
        if int4_group:
            q_layers.append(dict(qkv=PackedLinear.int4(qkv, int4_group), o=PackedLinear.int4(mats["wo"], int4_group),
                                 gu=PackedLinear.int4_pair(mats["w_gate"], mats["w_up"], int4_group),
                                 down=PackedLinear.int4(mats["w_down"], int4_group)))
        del qkv
    common = dict(embedding=embedding, attn_norms=attn_norms, mlp_norms=mlp_norms, final_norm=final_norm, rope=rope)
    fw = DeviceWeights(geo, f_layers, PackedLinear.f16(lm_head), wmode=_lib.W_F16, **common) if want_fp16 else None
    qw = None
    if int4_group:
        qw = DeviceWeights(geo, q_layers, PackedLinear.int4(lm_head, int4_group), wmode=_lib.W_INT4, **common)
    return fw, qw


# ---------------------------------------------------------------------------
# launch planning
# ---------------------------------------------------------------------------


def plan_attention_splits(n_heads_total: int, max_chunks: int, ctas_per_sm: int = 2) -> int:
    """Main-region splits per head so every main CTA is resident in one wave
    (the two short tail CTAs per head are scheduled after them)."""
    slots = ctas_per_sm * SM_COUNT
    heads = max(1, n_heads_total)
    best, best_eff = 1, -1.0
    for waves in (1, 2):  # each extra wave pays one more pipeline fill
        n = max(1, (waves * slots) // heads)
        if waves > 1 and max_chunks < 64 * n:
            # short contexts: CTAs of < 64 chunks cannot amortise a second wave's ring fill + merge
            # (verify at 32K: 4 splits 57.9 us vs 9 splits 62.6 us; 16K 34.3 vs 41.8; 128K keeps 9)
            break
        eff = (n * heads) / (math.ceil(n * heads / slots) * slots)
        if eff > best_eff + 0.05:
            best, best_eff = n, eff
    return max(1, min(best, max_chunks))


# ---------------------------------------------------------------------------
# forward runner
# ---------------------------------------------------------------------------


class Runner:
    """Scratch buffers + kernel sequence for forwards against one cache.

    Token buffer ``tok`` is [B][TS] (TS = max_T + 1): column 0 holds each sequence's pending
    token, columns 1.. its drafts; a forward over T rows reads columns [col, col + T).
    """

    def __init__(self, geo: Geometry, cache, *, max_cols: int = 16, attn_splits: int | None = None,
                 shard: tuple | None = None, gather=None):
        """``shard=(rank, world, process_group)``: KV-head sharding for a single sequence
        whose context does not fit one GPU.  This rank's cache and QKV
        weights hold heads [rank*H/world, (rank+1)*H/world); attention runs on those
        heads only and every rank needs all heads' rows before the replicated output
        projection / MLP.  ``gather``: None = torch.distributed.all_gather + prep (the
        collective baseline); "ipc" = the fused all-gather (the attention merge stores each
        head's f16 row into every rank's buffer over NVLink P2P, qs_gather_args), buffers
        exchanged as CUDA IPC handles over ``process_group``; or a parallel.HeadGather the
        caller links (ranks sharing one process, one stream each)."""
        torch = _torch()
        self.geo = geo
        self.cache = cache
        self.B = cache.batch
        if max_cols > _lib.MAX_COLS:
            raise ConfigError(f"{max_cols} activation rows exceed the linear kernels' {_lib.MAX_COLS}")
        self.max_cols = max_cols
        self.shard = shard
        if shard is not None:
            _, world, _ = shard
            if geo.num_kv_heads % world:
                raise ConfigError(f"{geo.num_kv_heads} KV heads do not shard over {world} ranks")
            lgeo = dataclasses.replace(geo, num_heads=geo.num_heads // world, num_kv_heads=geo.num_kv_heads // world)
        else:
            lgeo = geo
        self.lgeo = lgeo  # this rank's attention heads
        dev = torch.device("cuda")
        d, nq = geo.hidden, geo.nq
        self.x = torch.zeros((max_cols, d), dtype=torch.float32, device=dev)
        self.q = torch.zeros((max_cols, lgeo.nq), dtype=torch.float32, device=dev)
        self.attn = torch.zeros_like(self.q)
        if shard is not None:
            self.attn_full = torch.zeros((max_cols, nq), dtype=torch.float32, device=dev)
            self.gather_bufs = [torch.zeros((max_cols, lgeo.nq), dtype=torch.float32, device=dev)
                                for _ in range(shard[1])]
        # f16 linear-layer inputs (+ 16-element sums for the INT4 zero-point term), padded rows
        kmax = max(d, nq)
        self.xh = torch.zeros((max_cols, (kmax + 64 + 7) // 8 * 8), dtype=torch.float16, device=dev)
        self.xs = torch.zeros((max_cols, (kmax // 16 + 8 + 3) // 4 * 4), dtype=torch.float32, device=dev)
        m = geo.mlp_hidden
        self.hh = torch.zeros((max_cols, (m + 64 + 7) // 8 * 8), dtype=torch.float16, device=dev)
        self.hs = torch.zeros((max_cols, (m // 16 + 8 + 3) // 4 * 4), dtype=torch.float32, device=dev)
        self.logits = torch.zeros((max_cols, geo.vocab), dtype=torch.float32, device=dev)
        self.max_T = max(1, max_cols // self.B)
        self.TS = self.max_T + 1
        self.tok = torch.zeros((self.B, self.TS), dtype=torch.int32, device=dev)
        self.amax = torch.zeros(max_cols, dtype=torch.int32, device=dev)
        self.res = torch.zeros(2 * self.B, dtype=torch.int32, device=dev)
        self.is_fp = not hasattr(cache, "d_n_blocks")
        self.flags = cache.d_flags
        r = lgeo.num_heads // lgeo.num_kv_heads
        self.r = r
        self._attn_splits_override = attn_splits
        ncols_q = self.max_T * r
        # query-column groups per KV head: <= 24 queries per CTA in the quantised target view (three
        # 8-query MMA tiles with TMEM-parked accumulators: a GQA verify reads each chunk once for all
        # its r*T queries), <= 12 in the draft / fp16 views
        self.n_qgroups_max = max(1, -(-ncols_q // 12))
        self._lin_cache: dict = {}
        self._gen = None
        self.gather = None
        if gather is not None:
            if shard is None:
                raise ConfigError("a fused gather needs shard=(rank, world, group)")
            from .parallel import HeadGather

            rank, world, group = shard
            if isinstance(gather, str):
                import torch.distributed as dist

                if world == 1 and not (dist.is_available() and dist.is_initialized()):
                    gather = HeadGather(1, 0, max_cols, self.xh.shape[1], self.xs.shape[1])
                else:
                    gather = HeadGather.exchange(world, rank, max_cols, self.xh.shape[1], self.xs.shape[1], group)
            if (gather.rows, gather.ld_h, gather.ld_s) != (max_cols, self.xh.shape[1], self.xs.shape[1]):
                raise ConfigError("gather buffers do not match the runner's activation rows")
            self.gather = gather
        self._plan()

    def _plan(self) -> None:
        """Capacity-dependent launch plan (re-run when the cache reallocates): split-K grid per
        view -- fixed for every T, so row results are batch-invariant (a T-row verify == T
        single-row steps, bit for bit) -- and the partials scratch it needs."""
        torch = _torch()
        cache = self.cache
        if self.is_fp:
            self.max_chunks = -(-cache.capacity // 64)
        else:
            self.max_chunks = -(-cache.max_blocks * cache.layout.group_size // 128)
        self._splits: dict = {}
        # queries per CTA (qs_attn_partials_floats): <= 24 in the target view, <= 12 in the draft / fp16
        # views (the target's groups of 24 are never more numerous than the groups of 12)
        nq_cta = 24
        max_splits = self._attn_splits_override or max(1, min(self.max_chunks, 4 * SM_COUNT))
        nparts = self.B * self.lgeo.num_kv_heads * self.n_qgroups_max * (max_splits + 2) * nq_cta * (self.geo.head_dim + 2)
        self.partials = torch.zeros(nparts, dtype=torch.float32, device="cuda")
        self.attn_counters = torch.zeros(self.B * self.lgeo.num_kv_heads * self.n_qgroups_max, dtype=torch.int32,
                                         device="cuda")
        self.fp_cps = 0
        if self.is_fp:
            self.fp_cps = -(-self.max_chunks // self.splits_for(_lib.VIEW_FP16))
        self._lin_cache.clear()
        self._gen = cache.generation

    def sync_generation(self) -> None:
        if self._gen != self.cache.generation:
            self._plan()

    def splits_for(self, view: int) -> int:
        """Main-region splits of the attention grid for one view (cached)."""
        n = self._splits.get(view)
        if n is None:
            if self._attn_splits_override:
                n = self._attn_splits_override
            else:
                cols = self.r if view == _lib.VIEW_DRAFT else min(24 if view == _lib.VIEW_TARGET else 12,
                                                                  self.max_T * self.r)
                occ = _lib.load().qs_attn_occupancy(self.geo.head_dim, cols, view)
                occ = occ if occ > 0 else 1
                # per-sequence, per-head plan -- never scaled by the batch, the rows per sequence or the
                # query groups -- so a sequence's rows are bit-identical whatever batch it decodes in
                # (batch-3 == three batch-1 runs) and a T-row verify equals T one-row target steps
                n = plan_attention_splits(self.lgeo.num_kv_heads, self.max_chunks, occ)
            self._splits[view] = n
        return n

    # -- linear ---------------------------------------------------------------
    def _fuse_prep(self, pl: PackedLinear, ncols: int) -> bool:
        """Single-row steps build their f16 input (+ RMS norm) in the linear kernel (no
        qs_prep_act launch); both run act_prep_row, so the bits are the same either way."""
        return ncols == 1 and pl.K <= 4096

    def _linear(self, pl: PackedLinear, src, y, ncols: int, epi: int, *, ldy: int | None = None, layer: int = 0,
                T: int = 1, row_offset: int = 0, yh=None, stream: int, xf=None, gain=None) -> None:
        """One persistent linear launch.  ``src`` = (f16 rows, 16-sums) written by
        ``qs_prep_act`` or a SiLU epilogue; ``yh`` = (f16 rows, 16-sums) output
        of the SiLU epilogue."""
        key = (id(pl), ncols, epi, layer, T, row_offset, xf is not None)
        a = self._lin_cache.get(key)
        if a is None:
            geo = self.geo
            a = _lib.LinearArgs()
            a.wmode, a.epi, a.N, a.K, a.ncols = pl.wmode, epi, pl.N, pl.K, ncols
            a.wgroup = pl.group if pl.wmode == _lib.W_INT4 else 16
            a.w = pl.w.data_ptr()
            a.wparams = pl.params.data_ptr() if pl.params is not None else None
            xh, xs = src
            a.xh, a.ldxh = xh.data_ptr(), xh.shape[1]
            a.xs, a.ldxs = xs.data_ptr(), xs.shape[1]
            a.y = y.data_ptr() if y is not None else None
            a.ldy = ldy if ldy is not None else (y.shape[1] if y is not None else 0)
            if yh is not None:
                a.yh, a.ldyh = yh[0].data_ptr(), yh[0].shape[1]
                a.ys, a.ldys = yh[1].data_ptr(), yh[1].shape[1]
            if xf is not None:
                a.xf, a.ldxf = xf.data_ptr(), xf.shape[1]
                a.gain = gain.data_ptr() if gain is not None else None
                a.eps = float(geo.norm_eps)
            if epi == _lib.EPI_QKV:
                c = self.cache
                a.Nq, a.Nk, a.hd, a.T = self.lgeo.nq, self.lgeo.nk, geo.head_dim, T
                a.q_out = self.q.data_ptr()
                a.row_offset = row_offset
                a.rope = self._rope.data_ptr()
                a.max_pos = int(self._rope.shape[0])
                a.flags = self.flags.data_ptr()
                if self.is_fp:
                    L, H, cap, hd = c.num_layers, c.kv_heads, c.capacity, c.head_dim
                    a.k_dst = c.k[0, layer].data_ptr()
                    a.v_dst = c.v[0, layer].data_ptr()
                    a.kv_seq_stride = L * H * cap * hd
                    a.kv_head_stride = cap * hd
                    a.row_cap = cap
                    a.row_base = c.d_len.data_ptr()
                    a.pos_base = c.d_len.data_ptr()
                else:
                    lay = c.layout
                    L, H, hd, R = lay.num_layers, lay.kv_heads, lay.head_dim, c.fp_rows
                    a.k_dst = c.fp_k[0, layer, 1].data_ptr()
                    a.v_dst = c.fp_v[0, layer, 1].data_ptr()
                    a.kv_seq_stride = L * 2 * H * R * hd
                    a.kv_head_stride = R * hd
                    a.row_cap = R
                    a.row_base = c.d_fp2_len.data_ptr()
                    a.pos_base = c.d_pos.data_ptr()
            self._lin_cache[key] = a
        _lib.check(_lib.load().qs_linear(a, stream), "qs_linear")

    def _prep(self, x, gain, dst, ncols: int, stream: int) -> None:
        xh, xs = dst
        _lib.check(_lib.load().qs_prep_act(x.data_ptr(), gain.data_ptr() if gain is not None else None,
                                           float(self.geo.norm_eps), xh.data_ptr(), xh.shape[1], xs.data_ptr(),
                                           xs.shape[1], ncols, x.shape[1], stream), "qs_prep_act")

    # -- attention --------------------------------------------------------------
    def _attention(self, layer: int, view: int, T: int, row_offset: int, stream: int) -> None:
        key = ("attn", layer, view, T, row_offset)
        a = self._lin_cache.get(key)
        if a is None:
            geo, c = self.geo, self.cache
            a = _lib.AttnArgs()
            a.B, a.Hkv, a.hd, a.T, a.r = self.B, self.lgeo.num_kv_heads, geo.head_dim, T, self.r
            a.n_queries = T * self.r
            quant_target = view == _lib.VIEW_TARGET and not self.is_fp and layer not in getattr(
                self.cache.layout, "sensitive_layers", ())
            a.n_qgroups = max(1, -(-a.n_queries // (_TGT_GROUP if quant_target else 12)))
            a.n_main = self.splits_for(view if not self.is_fp else _lib.VIEW_FP16)
            a.row_offset = row_offset
            a.sm_scale_log2 = float(1.4426950408889634 / math.sqrt(geo.head_dim))
            a.q, a.out, a.q_row_stride = self.q.data_ptr(), self.attn.data_ptr(), self.lgeo.nq
            a.partials, a.counters = self.partials.data_ptr(), self.attn_counters.data_ptr()
            # fused hand-off: the merge writes the O projection's f16 input + 16-sums (no prep launch);
            # a head shard gathers first, so its merge writes only the f32 rows
            if self.shard is None or self.gather is not None:
                a.out_h, a.ld_out_h = self.xh.data_ptr(), self.xh.shape[1]
                a.out_s, a.ld_out_s = self.xs.data_ptr(), self.xs.shape[1]
            if self.gather is not None:
                rank, world, _ = self.shard
                self.gather.fill(a, arrivals=world * self.B * a.Hkv * a.n_qgroups, q_col_offset=rank * self.lgeo.nq)
            if self.is_fp:
                a.G = 64
                a.fp_len = c.d_len.data_ptr()
                a.main_is_fpcache, a.fpcache_cps = 1, self.fp_cps
                a.main_k, a.main_v = c.k[0, layer].data_ptr(), c.v[0, layer].data_ptr()
                a.main_seq_stride = c.num_layers * c.kv_heads * c.capacity * c.head_dim
                a.main_head_stride = c.capacity * c.head_dim
                mode = _lib.VIEW_FP16
            else:
                lay = c.layout
                L, H, G, hd, MB = lay.num_layers, lay.kv_heads, lay.group_size, lay.head_dim, c.max_blocks
                a.G = G
                a.n_blocks, a.fp1_len, a.fp2_len = c.d_n_blocks.data_ptr(), c.d_fp1_len.data_ptr(), c.d_fp2_len.data_ptr()
                a.fp1_k, a.fp1_v = c.fp_k[0, layer, 0].data_ptr(), c.fp_v[0, layer, 0].data_ptr()
                a.fp2_k, a.fp2_v = c.fp_k[0, layer, 1].data_ptr(), c.fp_v[0, layer, 1].data_ptr()
                a.fp_seq_stride = L * 2 * H * c.fp_rows * hd
                a.fp_rows = c.fp_rows
                if layer in lay.sensitive_layers:
                    slot = c._sens.index(layer)
                    a.main_k, a.main_v = c.arch_k[0, slot].data_ptr(), c.arch_v[0, slot].data_ptr()
                    a.main_seq_stride = len(c._sens) * H * MB * G * hd
                    a.main_head_stride = MB * G * hd
                    mode = _lib.VIEW_FP16
                else:
                    pb = G * hd // 2
                    a.ku, a.kl = c.ku[0, layer].data_ptr(), c.kl[0, layer].data_ptr()
                    a.vu, a.vl = c.vu[0, layer].data_ptr(), c.vl[0, layer].data_ptr()
                    a.plane_seq_stride = L * H * MB * pb
                    a.plane_head_stride = MB * pb
                    a.kp, a.vp = c.kp[0, layer].data_ptr(), c.vp[0, layer].data_ptr()
                    a.kp_seq_stride, a.kp_head_stride = L * H * MB * hd, MB * hd
                    a.vp_seq_stride, a.vp_head_stride = L * H * MB * G, MB * G
                    mode = view
            self._lin_cache[key] = (a, mode)
        else:
            a, mode = a
        _lib.check(_lib.load().qs_attn_decode(a, mode, stream), "qs_attn_decode")

    # -- full forward -------------------------------------------------------------
    def forward(self, w: DeviceWeights, T: int, view: int, *, row_offset: int = 0, tok_col: int = 0,
                argmax_to=None, stream=None) -> None:
        """Run one forward over ``T`` rows per sequence reading tokens ``tok[:, tok_col:tok_col+T]``;
        logits land in ``self.logits[:B*T]`` (row b*T + t).  ``argmax_to = (ptr, stride)`` stores
        each row's argmax at ptr[row * stride]."""
        geo = self.geo
        self.sync_generation()
        s = _lib.stream_ptr(stream)
        lib = _lib.load()
        ncols = self.B * T
        if ncols > self.max_cols or tok_col + T > self.TS:
            raise ConfigError(f"forward of {self.B} x {T} rows exceeds runner capacity {self.max_cols}")
        self._rope = w.rope
        d = geo.hidden
        tok_ptr = self.tok.data_ptr() + 4 * tok_col
        _lib.check(lib.qs_embed(w.embedding.data_ptr(), tok_ptr, self.TS, T, self.x.data_ptr(), ncols, d, geo.vocab,
                                self.flags.data_ptr(), s), "qs_embed")
        X, H = (self.xh, self.xs), (self.hh, self.hs)
        for li, lw in enumerate(w.layers):
            if self._fuse_prep(lw["qkv"], ncols):
                self._linear(lw["qkv"], X, None, ncols, _lib.EPI_QKV, layer=li, T=T, row_offset=row_offset, stream=s,
                             xf=self.x, gain=w.attn_norms[li])
            else:
                self._prep(self.x, w.attn_norms[li], X, ncols, s)
                self._linear(lw["qkv"], X, None, ncols, _lib.EPI_QKV, layer=li, T=T, row_offset=row_offset, stream=s)
            self._attention(li, view, T, row_offset, s)  # also writes X = (f16, 16-sums) of its output
            if self.shard is not None and self.gather is None:
                self._gather_heads(ncols)
                self._prep(self.attn_full, None, X, ncols, s)
            self._linear(lw["o"], X, self.x, ncols, _lib.EPI_ADD, stream=s)
            if self._fuse_prep(lw["gu"], ncols):
                self._linear(lw["gu"], X, None, ncols, _lib.EPI_SILU_MUL, yh=H, stream=s, xf=self.x,
                             gain=w.mlp_norms[li])
            else:
                self._prep(self.x, w.mlp_norms[li], X, ncols, s)
                self._linear(lw["gu"], X, None, ncols, _lib.EPI_SILU_MUL, yh=H, stream=s)
            self._linear(lw["down"], H, self.x, ncols, _lib.EPI_ADD, stream=s)
        if self._fuse_prep(w.lm_head, ncols):
            self._linear(w.lm_head, X, self.logits, ncols, _lib.EPI_STORE, stream=s, xf=self.x, gain=w.final_norm)
        else:
            self._prep(self.x, w.final_norm, X, ncols, s)
            self._linear(w.lm_head, X, self.logits, ncols, _lib.EPI_STORE, stream=s)
        if argmax_to is not None:
            ptr, stride = argmax_to if isinstance(argmax_to, tuple) else (argmax_to, 1)
            _lib.check(lib.qs_argmax(self.logits.data_ptr(), ncols, geo.vocab, ptr, stride, s), "qs_argmax")

    def _gather_heads(self, ncols: int) -> None:
        """All-gather every rank's attention rows [ncols, H_local*hd] into [ncols, H*hd]
        (rank r's heads are the r-th block of the head order)."""
        import torch.distributed as dist

        _, world, group = self.shard
        nql = self.lgeo.nq
        bufs = [b[:ncols] for b in self.gather_bufs]
        dist.all_gather(bufs, self.attn[:ncols].contiguous(), group=group)
        full = self.attn_full[:ncols].view(ncols, world, nql)
        for r in range(world):
            full[:, r].copy_(bufs[r])

    def kernel_launches_per_forward(self, nlayers: int, fused_prep: bool = False) -> int:
        """embed + per layer (prep, QKV, attention, O, prep, gate/up, down) + prep, lm_head, argmax;
        single-row steps build their inputs in-kernel (``fused_prep``: no prep launches)."""
        return 1 + nlayers * (5 if fused_prep else 7) + (2 if fused_prep else 3)
