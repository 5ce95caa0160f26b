"""Llama-style decoder API on the B200 runtime.

Mirrors /root/reference/pkg/src/quantspec/model.py: ModelConfig, ModelWeights,
init_weights, quantize_model_weights, prefill, decode_step, chunked_attention
and StepCost keep the reference names, arguments and errors.  Compute runs in
the sm_100a kernels (runtime.py); host NumPy weights are uploaded once and
cached on the ModelWeights object.

Extensions: ``num_kv_heads`` (GQA) and ``verify_step`` (T rows in one
forward -- the batched form of the gamma+1 sequential target steps of
Q/specdec.py:270-273).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib, qspw, quant
from .cache import CacheLayout, CacheView, FpKVCache, HierarchicalKVCache
from .errors import BufferOverflowError, ConfigError, DataError, DimensionError, EmptyPromptError, FormatError
from .runtime import DeviceWeights, Geometry, Runner, build_device_weights, rope_table

F32_BYTES = 4.0
INT4_BYTES = 0.5
DTYPE = np.float32

# Q/roofline.py:32-34 (flop model used by StepCost)
SOFTMAX_FLOPS_PER_SCORE = 5.0
NORM_FLOPS_PER_ELEM = 4.0
ACT_FLOPS_PER_ELEM = 4.0


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise ConfigError("the B200 model path needs a CUDA device (no CPU fallback)")
    return torch


@dataclass(frozen=True)
class ModelConfig:
    num_layers: int
    num_heads: int
    head_dim: int
    hidden: int
    mlp_hidden: int
    vocab: int
    max_positions: int
    rope_base: float = 10000.0
    norm_eps: float = 1e-5
    num_kv_heads: int | None = None

    def __post_init__(self) -> None:
        if self.hidden != self.num_heads * self.head_dim:
            raise ConfigError(
                f"hidden ({self.hidden}) must equal num_heads*head_dim ({self.num_heads}*{self.head_dim})"
            )
        if self.vocab < 2:
            raise ConfigError(f"vocab must be >= 2, got {self.vocab}")
        if min(self.num_layers, self.mlp_hidden, self.max_positions) < 1:
            raise ConfigError("model dimensions must be positive")
        if self.num_kv_heads is not None and self.num_heads % self.num_kv_heads:
            raise ConfigError("num_heads must be a multiple of num_kv_heads")

    @property
    def kv_heads(self) -> int:
        return self.num_kv_heads or self.num_heads

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim

    def geometry(self) -> Geometry:
        return Geometry(self.num_layers, self.hidden, self.num_heads, self.kv_heads, self.head_dim, self.mlp_hidden,
                        self.vocab, self.max_positions, self.rope_base, self.norm_eps)


@dataclass
class LayerWeights:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w_gate: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray
    attn_norm: np.ndarray
    mlp_norm: np.ndarray


_MATS = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")


@dataclass
class ModelWeights:
    config: ModelConfig
    embedding: np.ndarray
    layers: list
    final_norm: np.ndarray
    lm_head: np.ndarray
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    def named_tensors(self):
        yield "embedding", self.embedding
        for i, lw in enumerate(self.layers):
            for name in _MATS + ("attn_norm", "mlp_norm"):
                yield f"layers.{i}.{name}", getattr(lw, name)
        yield "final_norm", self.final_norm
        yield "lm_head", self.lm_head

    def device(self, int4_group: int | None = None):
        """(fp16 DeviceWeights, INT4 DeviceWeights or None), uploaded once."""
        torch = _torch()
        key = ("fp16",)
        if key not in self._device:
            cfg = self.config
            geo = cfg.geometry()
            rope = rope_table(cfg.head_dim, cfg.rope_base, cfg.max_positions)
            emb = torch.from_numpy(np.ascontiguousarray(self.embedding, dtype=np.float32)).cuda()
            an = [torch.from_numpy(np.ascontiguousarray(lw.attn_norm, dtype=np.float32)).cuda() for lw in self.layers]
            mn = [torch.from_numpy(np.ascontiguousarray(lw.mlp_norm, dtype=np.float32)).cuda() for lw in self.layers]
            fn = torch.from_numpy(np.ascontiguousarray(self.final_norm, dtype=np.float32)).cuda()
            head = torch.from_numpy(np.ascontiguousarray(self.lm_head, dtype=np.float32)).cuda()

            def mats():
                for lw in self.layers:
                    yield {n: torch.from_numpy(np.ascontiguousarray(getattr(lw, n), dtype=np.float32)).cuda() for n in _MATS}

            fw, _ = build_device_weights(geo, mats(), emb, fn, head, an, mn, rope=rope)
            self._device[key] = fw
        fw = self._device[key]
        qw = None
        if int4_group:
            qkey = ("int4", int4_group)
            if qkey not in self._device:
                head = torch.from_numpy(np.ascontiguousarray(self.lm_head, dtype=np.float32)).cuda()

                def mats():
                    for lw in self.layers:
                        yield {n: torch.from_numpy(np.ascontiguousarray(getattr(lw, n), dtype=np.float32)).cuda() for n in _MATS}

                _, qw = build_device_weights(fw.geo, mats(), fw.embedding, fw.final_norm, head, fw.attn_norms,
                                             fw.mlp_norms, int4_group=int4_group, rope=fw.rope, want_fp16=False)
                self._device[qkey] = qw
            qw = self._device[qkey]
        return fw, qw


def init_weights(config: ModelConfig, seed: int = 0) -> ModelWeights:
    """Seeded random weights with 1/sqrt(fan_in) scaling (Q/model.py:89-117 draw order)."""
    rng = np.random.default_rng(seed)
    d, m, v = config.hidden, config.mlp_hidden, config.vocab
    kvd = config.kv_dim

    def mat(rows, cols):
        return (rng.standard_normal((rows, cols)) / np.sqrt(rows)).astype(DTYPE)

    layers = [
        LayerWeights(wq=mat(d, d), wk=mat(d, kvd), wv=mat(d, kvd), wo=mat(d, d), w_gate=mat(d, m), w_up=mat(d, m),
                     w_down=mat(m, d), attn_norm=np.ones(d, DTYPE), mlp_norm=np.ones(d, DTYPE))
        for _ in range(config.num_layers)
    ]
    return ModelWeights(config=config, embedding=rng.standard_normal((v, d)).astype(DTYPE), layers=layers,
                        final_norm=np.ones(d, DTYPE), lm_head=mat(d, v))


@dataclass
class QuantizedModelWeights:
    """Draft weight set: INT4 planes (reference packing) + device frag4 copies."""

    config: ModelConfig
    planes: dict
    group_size: int
    int4_weight_bytes: float
    device: DeviceWeights | None = None

    @property
    def lm_head(self) -> np.ndarray:
        return quant.dequantize_weights(self.planes["lm_head"])


def quantize_model_weights(weights: ModelWeights, group_size: int) -> QuantizedModelWeights:
    """Q/model.py:141-168: every projection and lm_head to INT4 (embedding/norms stay fp)."""
    planes = {}
    total = 0.0
    for i, lw in enumerate(weights.layers):
        for name in _MATS:
            q = quant.quantize_weights(getattr(lw, name), group_size)
            planes[f"layers.{i}.{name}"] = q
            total += q.code_bytes()
    qh = quant.quantize_weights(weights.lm_head, group_size)
    planes["lm_head"] = qh
    total += qh.code_bytes()
    _, qw = weights.device(int4_group=group_size)
    return QuantizedModelWeights(weights.config, planes, group_size, total, qw)


@dataclass
class StepCost:
    """Per-step modeled load/compute accounting (Q/model.py:230-251)."""

    flops: float = 0.0
    weight_bytes: float = 0.0
    kv_quantized_bytes: float = 0.0
    kv_param_bytes: float = 0.0
    kv_fp_bytes: float = 0.0
    kv_quantized_elements: int = 0

    @property
    def total_bytes(self) -> float:
        return self.weight_bytes + self.kv_quantized_bytes + self.kv_param_bytes + self.kv_fp_bytes

    def add(self, other: "StepCost") -> None:
        self.flops += other.flops
        self.weight_bytes += other.weight_bytes
        self.kv_quantized_bytes += other.kv_quantized_bytes
        self.kv_param_bytes += other.kv_param_bytes
        self.kv_fp_bytes += other.kv_fp_bytes
        self.kv_quantized_elements += other.kv_quantized_elements


def _weight_elem_count(cfg: ModelConfig) -> int:
    d, m, v = cfg.hidden, cfg.mlp_hidden, cfg.vocab
    return cfg.num_layers * (2 * d * d + 2 * d * cfg.kv_dim + 3 * d * m) + d * v


# ---------------------------------------------------------------------------
# runners are cached per (cache object) so repeated decode_step calls reuse
# scratch buffers and prepared launch arguments
# ---------------------------------------------------------------------------

_RUNNERS: dict = {}


def runner_for(cfg: ModelConfig, cache, max_cols: int = 16) -> Runner:
    key = id(cache)
    r = _RUNNERS.get(key)
    if r is None or r.cache is not cache or r.max_cols < max_cols:
        if len(_RUNNERS) > 64:
            _RUNNERS.clear()
        r = Runner(cfg.geometry(), cache, max_cols=max(max_cols, 16))
        _RUNNERS[key] = r
    return r


def _view_kind(cache, view: str) -> int:
    if isinstance(cache, FpKVCache):
        return _lib.VIEW_FP16
    return {"draft": _lib.VIEW_DRAFT, "target": _lib.VIEW_TARGET}[view]


def modeled_view_cost(cache, view: str, cfg: ModelConfig, t_ctx_after: int, seq: int = 0) -> StepCost:
    """Per-forward modeled bytes/flops exactly as decode_step accumulates them."""
    c = StepCost()
    d, m = cfg.hidden, cfg.mlp_hidden
    for layer in range(cfg.num_layers):
        qb, pb, fb, qe = _view_bytes(cache, layer, view, seq)
        c.kv_quantized_bytes += qb
        c.kv_param_bytes += pb
        c.kv_fp_bytes += fb
        c.kv_quantized_elements += qe
        c.flops += 2.0 * (2 * d * d + 2 * d * cfg.kv_dim + 3 * d * m)
        c.flops += 4.0 * t_ctx_after * d
        c.flops += SOFTMAX_FLOPS_PER_SCORE * t_ctx_after * cfg.num_heads
        c.flops += NORM_FLOPS_PER_ELEM * 2 * d + ACT_FLOPS_PER_ELEM * m
    c.flops += 2.0 * d * cfg.vocab + NORM_FLOPS_PER_ELEM * d
    return c


def _view_bytes(cache, layer: int, view: str, seq: int = 0):
    """CacheView byte fields (Q/cache.py:345-378) from the host length mirror."""
    if isinstance(cache, FpKVCache):
        n = int(cache._lens[seq, layer])
        return 0.0, 0.0, 4.0 * 2 * n * cache.kv_dim, 0
    lay = cache.layout
    nq = int(cache._nq[seq])
    qb = pb = fb = 0.0
    qe = 0
    if layer in lay.sensitive_layers:
        fb += 4.0 * 2 * nq * lay.kv_dim
    elif nq:
        qe = 2 * nq * lay.kv_dim
        qb = (0.5 if view == "draft" else 1.0) * qe
        groups = cache._groups_per_block() * (nq // lay.group_size)
        pb = 8.0 * groups * (2 if view == "target" else 1)
    for n in (int(cache._fp1[seq]), int(cache._fp2[seq, layer])):
        fb += 4.0 * 2 * n * lay.kv_dim
    return qb, pb, fb, qe


def _validate_step(weights: ModelWeights, token: int, cache, view: str, weight_mode: str, draft_weights):
    cfg = weights.config
    if not 0 <= int(token) < cfg.vocab:
        raise DataError(f"token id {token} outside vocab {cfg.vocab}")
    if cache.seq_len == 0:
        raise ConfigError("decode requires a prefilled cache")
    if weight_mode not in ("fp", "int4"):
        raise ConfigError(f"unknown weight mode {weight_mode!r}")
    if weight_mode == "int4":
        if draft_weights is None:
            raise ConfigError("weight_mode='int4' requires quantized draft weights")
        if view != "draft":
            raise ConfigError("INT4 weights are only used on the draft view")
    if view not in ("fp", "draft", "target"):
        raise ConfigError(f"cache {type(cache).__name__} does not provide a {view!r} view")
    if view == "fp" and not isinstance(cache, FpKVCache):
        raise ConfigError(f"cache {type(cache).__name__} does not provide a {view!r} view")


def decode_step(weights: ModelWeights, token: int, cache, *, view: str = "fp", weight_mode: str = "fp",
                draft_weights: QuantizedModelWeights | None = None):
    """One decode pass: append the token's K/V, attend over ``view``, return logits (Q/model.py:324-407)."""
    logits, cost = verify_step(weights, [token], cache, view=view, weight_mode=weight_mode, draft_weights=draft_weights)
    return logits[0], cost


def verify_step(weights: ModelWeights, tokens, cache, *, view: str = "target", weight_mode: str = "fp",
                draft_weights: QuantizedModelWeights | None = None):
    """T consecutive tokens in ONE forward (causal inside the new rows).

    Equivalent to T sequential decode_step calls (Q/specdec.py:270-273) but
    reads the KV store once; returns (f32 logits [T, V], summed StepCost).
    """
    torch = _torch()
    cfg = weights.config
    toks = [int(t) for t in tokens]
    for t in toks:
        _validate_step(weights, t, cache, view, weight_mode, draft_weights)
    T = len(toks)
    if cache.seq_len + T > cfg.max_positions:
        raise ConfigError(f"position {cache.seq_len + T - 1} exceeds max positions {cfg.max_positions}")
    if not isinstance(cache, FpKVCache) and cache.fp2_len + T > cache.layout.group_size:
        raise BufferOverflowError("fp2 is full; the engine must flush before appending")
    if getattr(cache, "batch", 1) != 1:
        raise ConfigError("decode_step / verify_step drive a single-sequence cache; batches run through SpecEngine")
    fw, _ = weights.device()
    w = draft_weights.device if weight_mode == "int4" else fw
    if isinstance(cache, FpKVCache):
        cache.ensure_tokens(cache.seq_len + T)  # grows like the reference's FpKVCache (Q/cache.py:606-612)
    run = runner_for(cfg, cache, T)
    run.tok[0, :T] = torch.tensor(toks, dtype=torch.int32, device="cuda")
    run.forward(w, T, _view_kind(cache, view))
    flags = int(run.flags.item())
    if flags:
        run.flags.zero_()
        if flags & _lib.FLAG_VOCAB:
            raise DataError("token id outside vocab")
        if flags & _lib.FLAG_POSITION:
            raise ConfigError(f"position beyond the rope table ({cfg.max_positions})")
        raise BufferOverflowError(f"device status {flags:#x}")
    logits = run.logits[:T].cpu().numpy().copy()
    cost = StepCost()
    wbytes = draft_weights.int4_weight_bytes if weight_mode == "int4" else F32_BYTES * _weight_elem_count(cfg)
    for i in range(T):
        # row i sees the rows 0..i appended by this call (as i+1 sequential steps would)
        c = modeled_view_cost(cache, view, cfg, cache.seq_len + i + 1)
        c.kv_fp_bytes += 4.0 * 2 * (i + 1) * cfg.kv_dim * cfg.num_layers
        c.weight_bytes = wbytes
        cost.add(c)
    cache._advance(T)
    return logits, cost


def prefill(weights: ModelWeights, tokens, cache_mode: str = "fp", *, group_size: int | None = None,
            sensitive_layers: frozenset = frozenset(), max_tokens: int | None = None):
    """Causal forward over the prompt; returns last-token logits and a device cache (Q/model.py:268-321)."""
    from ._prefill import prefill_device

    cfg = weights.config
    ids = np.asarray(tokens, dtype=np.int64).ravel()
    if ids.size == 0:
        raise EmptyPromptError("prompt must contain at least one token")
    if ids.size > cfg.max_positions:
        raise ConfigError(f"prompt of {ids.size} tokens exceeds max positions {cfg.max_positions}")
    if ids.min() < 0 or ids.max() >= cfg.vocab:
        raise DataError(f"token ids must lie in [0, {cfg.vocab})")
    if cache_mode not in ("fp", "hierarchical"):
        raise ConfigError(f"unknown cache mode {cache_mode!r}")
    return prefill_device(weights, ids, cache_mode, group_size=group_size, sensitive_layers=sensitive_layers,
                          max_tokens=max_tokens)


def prefill_batch(weights: ModelWeights, prompts, *, group_size: int | None = None,
                  sensitive_layers: frozenset = frozenset(), max_tokens: int | None = None):
    """Prefill independent prompts (any lengths) into one batched HierarchicalKVCache for the
    ragged-batch SpecEngine (config 4); returns (list of last-token logits, cache)."""
    from ._prefill import prefill_batch_device

    cfg = weights.config
    ps = [np.asarray(p, dtype=np.int64).ravel() for p in prompts]
    for ids in ps:
        if ids.size == 0:
            raise EmptyPromptError("prompt must contain at least one token")
        if ids.size > cfg.max_positions:
            raise ConfigError(f"prompt of {ids.size} tokens exceeds max positions {cfg.max_positions}")
        if ids.min() < 0 or ids.max() >= cfg.vocab:
            raise DataError(f"token ids must lie in [0, {cfg.vocab})")
    return prefill_batch_device(weights, ps, group_size=group_size, sensitive_layers=sensitive_layers,
                                max_tokens=max_tokens)


def chunked_attention(q: np.ndarray, chunks, scale: float | None = None) -> np.ndarray:
    """Single-head attention of ``q`` over (K, V) chunks (Q/model.py:198-222), on device (fp16 K/V)."""
    torch = _torch()
    q = np.asarray(q, dtype=DTYPE).ravel()
    if not chunks:
        raise ConfigError("chunked attention needs at least one chunk")
    dim = q.size
    ks, vs = [], []
    for k, v in chunks:
        k = np.asarray(k, dtype=DTYPE)
        v = np.asarray(v, dtype=DTYPE)
        if k.ndim != 2 or k.shape[1] != dim or v.shape != k.shape:
            raise DimensionError(f"chunk shapes {k.shape}/{v.shape} do not match head dim {dim}")
        ks.append(k)
        vs.append(v)
    kk = np.concatenate(ks)
    vv = np.concatenate(vs)
    if kk.shape[0] == 0:
        raise ConfigError("chunked attention needs at least one token")
    if scale is not None and abs(scale - 1.0 / math.sqrt(dim)) > 1e-12:
        q = q * np.float32(scale * math.sqrt(dim))
    n = kk.shape[0]
    cache = FpKVCache(1, dim, capacity=n + 1, head_dim=dim)
    cache.load_prefill_layer(0, kk[:-1] if n > 1 else kk[:0], vv[:-1] if n > 1 else vv[:0])
    cache.finish_prefill(n - 1)
    geo = Geometry(1, dim, 1, 1, dim, 16, 2, n + 1)
    run = Runner(geo, cache, max_cols=1)
    # place the query and the last row directly, then run the attention kernel only
    run.q[0, :dim] = torch.from_numpy(q).cuda()
    cache.k[0, 0, 0, n - 1] = torch.from_numpy(kk[-1]).cuda().half()
    cache.v[0, 0, 0, n - 1] = torch.from_numpy(vv[-1]).cuda().half()
    run._attention(0, _lib.VIEW_FP16, 1, 0, _lib.stream_ptr())
    return run.attn[0, :dim].cpu().numpy().copy()


# ---------------------------------------------------------------------------
# QSPW weight file (Q/model.py:415-524)
# ---------------------------------------------------------------------------


def save_weights(path, weights: ModelWeights) -> None:
    """Write the reference's QSPW weight file (Q/model.py:415-458; codec in qspw.py)."""
    cfg = weights.config
    dims = (cfg.num_layers, cfg.num_heads, cfg.head_dim, cfg.hidden, cfg.mlp_hidden, cfg.vocab, cfg.max_positions)
    with open(path, "wb") as f:
        f.write(qspw.encode(dims, cfg.rope_base, cfg.norm_eps, weights.named_tensors()))


def load_weights(path) -> ModelWeights:
    """Read a QSPW weight file (Q/model.py:461-524): FormatError on a bad magic / version, truncation,
    checksum mismatch, a missing tensor or a wrong shape.  GQA files (this package's extension: the
    reference is MHA) carry their KV width in the wk / wv shapes."""
    with open(path, "rb") as f:
        dims, rope_base, norm_eps, tensors = qspw.decode(f.read())
    L, H, hd, d, mh, v, max_pos = dims
    wk = tensors.get("layers.0.wk")
    kvd = int(wk.shape[1]) if wk is not None and wk.ndim == 2 and wk.shape[1] % max(hd, 1) == 0 else d
    cfg = ModelConfig(L, H, hd, d, mh, v, max_pos, rope_base=rope_base, norm_eps=norm_eps,
                      num_kv_heads=None if kvd == d else kvd // hd)

    def grab(name, shape):
        a = tensors.get(name)
        if a is None:
            raise FormatError(f"weight file missing tensor {name!r}")
        if a.shape != shape:
            raise FormatError(f"tensor {name!r} has shape {a.shape}, expected {shape}")
        return a

    shapes = {"wq": (d, d), "wk": (d, kvd), "wv": (d, kvd), "wo": (d, d), "w_gate": (d, mh), "w_up": (d, mh),
              "w_down": (mh, d), "attn_norm": (d,), "mlp_norm": (d,)}
    layers = [LayerWeights(**{n: grab(f"layers.{i}.{n}", sh) for n, sh in shapes.items()}) for i in range(L)]
    return ModelWeights(cfg, grab("embedding", (v, d)), layers, grab("final_norm", (d,)), grab("lm_head", (d, v)))
