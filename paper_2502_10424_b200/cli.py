"""Experiment harness on the device path: run | gamma-sweep | ablate | gen-model.

Mirrors the reference CLI (/root/reference/pkg/src/quantspec/cli.py:233-284, 329-341): the same
configuration resolution (defaults <- JSON config file <- flags, cli.py:81-111), the same seeds
(model init seed + 2, prompt seed + 1, cli.py:118-139), the same output files (manifest.json,
metrics.csv, trace.ndjson, tokens.txt, gamma_sweep.csv, ablate.csv).  The reference's analytic
``modeled_speedup`` column (its roofline modeller is out of scope here) is replaced by
MEASURED numbers on the B200: decode tokens/s of the speculative run and of plain autoregressive
decoding over the same cache mode (prefill excluded, device time), and their ratio.

    python -m paper_2502_10424_b200 run --gamma 4 --out runs/a
    python -m paper_2502_10424_b200 gamma-sweep --gamma 1,2,4,6
    python -m paper_2502_10424_b200 ablate
"""

from __future__ import annotations

import argparse
import copy
import json
import sys
from pathlib import Path

import numpy as np

DEFAULT_CONFIG: dict = {
    "seed": 0,
    "out_dir": "runs/out",
    "model": {"num_layers": 2, "num_heads": 4, "head_dim": 16, "mlp_hidden": 176, "vocab": 64, "max_positions": 2048},
    "weights_path": None,
    "prompt": {"length": 384},
    "spec": {"gamma": 4, "decode_len": 90, "sampling": "greedy", "temperature": 1.0},
    "quant": {"kv_quant": True, "weight_quant": False, "group_size": 128, "weight_group_size": 32,
              "sensitive_layers": []},
}
ABLATION_MODES = (("neither", False, False), ("kv_only", True, False), ("weight_only", False, True),
                  ("both", True, True))
METRICS_HEADER = ["acceptance_rate", "mean_tokens_per_verification", "measured_tok_s", "measured_ar_tok_s",
                  "measured_speedup", "peak_cache_bytes", "drafted_tokens", "accepted_tokens", "verification_steps",
                  "emitted_tokens"]


def _merge(base: dict, over: dict) -> dict:
    out = copy.deepcopy(base)
    for k, v in over.items():
        out[k] = _merge(out[k], v) if isinstance(v, dict) and isinstance(out.get(k), dict) else copy.deepcopy(v)
    return out


def resolve_config(args) -> dict:
    cfg = copy.deepcopy(DEFAULT_CONFIG)
    if getattr(args, "config", None):
        cfg = _merge(cfg, json.loads(Path(args.config).read_text(encoding="utf-8")))
    if args.seed is not None:
        cfg["seed"] = args.seed
    if args.out is not None:
        cfg["out_dir"] = args.out
    if getattr(args, "kv_quant", None) is not None:
        cfg["quant"]["kv_quant"] = args.kv_quant
    if getattr(args, "weight_quant", None) is not None:
        cfg["quant"]["weight_quant"] = args.weight_quant
    if getattr(args, "decode_len", None) is not None:
        cfg["spec"]["decode_len"] = args.decode_len
    if getattr(args, "prompt_len", None) is not None:
        cfg["prompt"]["length"] = args.prompt_len
    return cfg


def _weights(cfg: dict):
    from . import model

    if cfg.get("weights_path"):
        return model.load_weights(cfg["weights_path"])
    m = cfg["model"]
    c = model.ModelConfig(num_layers=m["num_layers"], num_heads=m["num_heads"], head_dim=m["head_dim"],
                          hidden=m["num_heads"] * m["head_dim"], mlp_hidden=m["mlp_hidden"], vocab=m["vocab"],
                          max_positions=m["max_positions"], num_kv_heads=m.get("num_kv_heads"))
    return model.init_weights(c, seed=m.get("init_seed", cfg["seed"] + 2))


def _prompt(cfg: dict, vocab: int) -> np.ndarray:
    p = cfg["prompt"]
    return np.random.default_rng(p.get("seed", cfg["seed"] + 1)).integers(0, vocab, size=int(p["length"]),
                                                                          dtype=np.int64)


def _device_seconds(fn):
    import torch

    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out = fn()
    e.record()
    torch.cuda.synchronize()
    return out, s.elapsed_time(e) / 1e3


def run_experiment(cfg: dict) -> tuple:
    """One speculative decode (SpeculativeDecoder over the device engine) and the plain AR decode over
    the same cache mode; both timed on the device with the prefill excluded.  Returns
    (RunResult, spec tok/s, AR tok/s)."""
    from .engine import SpecEngine
    from .specdec import GREEDY, SpecConfig, SpeculativeDecoder, autoregressive_decode

    w = _weights(cfg)
    prompt = _prompt(cfg, w.config.vocab)
    s, q = cfg["spec"], cfg["quant"]
    spec = SpecConfig(gamma=int(s["gamma"]), decode_len=int(s["decode_len"]), sampling=s.get("sampling", GREEDY),
                      temperature=float(s.get("temperature", 1.0)), seed=int(cfg["seed"]),
                      weight_mode="int4" if q["weight_quant"] else "fp")
    kw = dict(kv_quant=bool(q["kv_quant"]), group_size=int(q["group_size"]),
              sensitive_layers=frozenset(q.get("sensitive_layers", [])))
    dec = SpeculativeDecoder(w, spec, weight_group_size=int(q.get("weight_group_size", 32)), **kw)
    if spec.sampling == GREEDY and kw["kv_quant"]:
        logits, cache = dec._prefill(prompt)
        fw, _ = w.device()
        dw = dec.draft_weights.device if dec.draft_weights is not None else fw
        eng = SpecEngine(fw, dw, cache, spec.gamma, max_positions=w.config.max_positions)
        res, dt = _device_seconds(lambda: dec.decode(eng, [int(np.argmax(logits))], decode_len=spec.decode_len)[0])
    else:  # host-decided paths (stochastic sampling, fp caches): timed end to end minus nothing
        res, dt = _device_seconds(lambda: dec.run(prompt))
    n_new = max(1, len(res.tokens) - 1)
    ar_kw = dict(kw, sampling=spec.sampling, temperature=spec.temperature, seed=spec.seed)
    _, dt_ar = _device_seconds(lambda: autoregressive_decode(w, prompt, int(s["decode_len"]), **ar_kw))
    return res, n_new / dt, n_new / dt_ar


def _row(m, tok_s, ar_tok_s) -> list:
    return [m.acceptance_rate, m.mean_tokens_per_verification, tok_s, ar_tok_s, tok_s / ar_tok_s, m.peak_cache_bytes,
            m.drafted_tokens, m.accepted_tokens, m.verification_steps, m.emitted_tokens]


def _csv(path: Path, header, rows) -> None:
    fmt = lambda v: repr(v) if isinstance(v, float) else str(v)  # noqa: E731
    path.write_text("\n".join([",".join(header)] + [",".join(fmt(v) for v in r) for r in rows]) + "\n",
                    encoding="utf-8")


def _manifest(out: Path, cfg: dict) -> None:
    (out / "manifest.json").write_text(json.dumps(cfg, sort_keys=True, indent=2) + "\n", encoding="utf-8")


def cmd_run(cfg: dict) -> int:
    out = Path(cfg["out_dir"])
    out.mkdir(parents=True, exist_ok=True)
    res, tok_s, ar = run_experiment(cfg)
    _manifest(out, cfg)
    _csv(out / "metrics.csv", METRICS_HEADER, [_row(res.metrics, tok_s, ar)])
    (out / "trace.ndjson").write_text(res.trace.to_ndjson(), encoding="utf-8")
    (out / "tokens.txt").write_text(" ".join(map(str, res.tokens)) + "\n", encoding="utf-8")
    print(f"acceptance {res.metrics.acceptance_rate:.4f}  {tok_s:.1f} tok/s  (AR {ar:.1f} tok/s, x{tok_s / ar:.2f})")
    return 0


def cmd_gamma_sweep(cfg: dict, gammas) -> int:
    out = Path(cfg["out_dir"])
    out.mkdir(parents=True, exist_ok=True)
    rows = []
    for g in sorted(set(int(x) for x in gammas)):
        sub = copy.deepcopy(cfg)
        sub["spec"]["gamma"] = g
        res, tok_s, ar = run_experiment(sub)
        rows.append([g, res.metrics.acceptance_rate, tok_s, tok_s / ar])
    best = max(range(len(rows)), key=lambda i: rows[i][2])
    _manifest(out, cfg)
    _csv(out / "gamma_sweep.csv", ["gamma", "acceptance_rate", "measured_tok_s", "measured_speedup", "best"],
         [r + [1 if i == best else 0] for i, r in enumerate(rows)])
    return 0


def cmd_ablate(cfg: dict) -> int:
    out = Path(cfg["out_dir"])
    out.mkdir(parents=True, exist_ok=True)
    rows = []
    for label, kv_q, w_q in ABLATION_MODES:
        sub = copy.deepcopy(cfg)
        sub["quant"]["kv_quant"], sub["quant"]["weight_quant"] = kv_q, w_q
        res, tok_s, ar = run_experiment(sub)
        rows.append([label, kv_q, w_q, res.metrics.acceptance_rate, tok_s, tok_s / ar])
    _manifest(out, cfg)
    _csv(out / "ablate.csv", ["mode", "kv_quant", "weight_quant", "acceptance_rate", "measured_tok_s",
                              "measured_speedup"], rows)
    return 0


def cmd_gen_model(cfg: dict) -> int:
    from . import model

    out = Path(cfg["out_dir"])
    out.mkdir(parents=True, exist_ok=True)
    model.save_weights(out / "weights.qspw", _weights(cfg))
    _manifest(out, cfg)
    return 0


def _bool(v: str) -> bool:
    if v.lower() in ("1", "true", "yes", "on"):
        return True
    if v.lower() in ("0", "false", "no", "off"):
        return False
    raise argparse.ArgumentTypeError(f"not a boolean: {v!r}")


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_2502_10424_b200")
    sub = p.add_subparsers(dest="cmd", required=True)
    for name, help_ in (("run", "one speculative decode experiment"), ("gamma-sweep", "repeat over a gamma list"),
                        ("ablate", "neither / kv_only / weight_only / both"), ("gen-model", "write seeded weights")):
        sp = sub.add_parser(name, help=help_)
        sp.add_argument("--config", default=None, help="JSON config file")
        sp.add_argument("--seed", type=int, default=None)
        sp.add_argument("--out", default=None, help="output directory")
        sp.add_argument("--kv-quant", dest="kv_quant", type=_bool, default=None)
        sp.add_argument("--weight-quant", dest="weight_quant", type=_bool, default=None)
        sp.add_argument("--decode-len", dest="decode_len", type=int, default=None)
        sp.add_argument("--prompt-len", dest="prompt_len", type=int, default=None)
        if name == "run":
            sp.add_argument("--gamma", type=int, default=None)
        if name == "gamma-sweep":
            sp.add_argument("--gamma", default="1,2,4,6", help="comma-separated list")
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    cfg = resolve_config(args)
    if args.cmd == "run":
        if args.gamma is not None:
            cfg["spec"]["gamma"] = args.gamma
        return cmd_run(cfg)
    if args.cmd == "gamma-sweep":
        return cmd_gamma_sweep(cfg, args.gamma.split(","))
    if args.cmd == "ablate":
        return cmd_ablate(cfg)
    return cmd_gen_model(cfg)


if __name__ == "__main__":
    sys.exit(main())
