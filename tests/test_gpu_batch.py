"""Ragged multi-sequence decode on one GPU (config 4's per-GPU batch).

Each sequence keeps the reference's own schedule inside the batch (Q/specdec.py:329-356:
gamma_step = min(gamma, fp2_space - 1, remaining) including the degenerate target-only step,
its own accepted count, its own flush of Q/cache.py:249-262).  Bars:
  * a batch-3 ragged run (different prompt lengths, so different fp2 fill levels and flush
    cycles) is token-identical to three batch-1 runs, and with fp16 draft weights (batch-invariant
    kernels end to end) its traces are identical too;
  * batch spec tokens == batch target-view AR tokens (greedy losslessness inside a batch);
  * per-sequence cache state after the run equals the oracle state machine driven with the
    same accept sequence.
"""

import numpy as np
import pytest

from oracle import qs_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2502_10424_b200 as qs  # noqa: E402

TOY = qs.ModelConfig(num_layers=2, num_heads=4, head_dim=16, hidden=64, mlp_hidden=176, vocab=64, max_positions=2048)
G = 16
CAP = 1024


@pytest.fixture(scope="module")
def toy():
    return qs.init_weights(TOY, seed=7)


def _decode(w, prompts, wm, decode_len, gamma=4):
    logits, cache = qs.prefill_batch(w, prompts, group_size=G, max_tokens=CAP)
    dec = qs.SpeculativeDecoder(w, qs.SpecConfig(gamma=gamma, decode_len=decode_len, weight_mode=wm), group_size=G)
    fw, _ = w.device()
    dw = dec.draft_weights.device if dec.draft_weights is not None else fw
    eng = qs.SpecEngine(fw, dw, cache, gamma)
    res = dec.decode(eng, [int(np.argmax(l)) for l in logits], decode_len=decode_len)
    return res, cache


PROMPTS = [np.random.default_rng(s).integers(0, 64, size=n) for s, n in ((21, 300), (22, 347), (23, 40))]


@pytest.mark.parametrize("wm", ["fp", "int4"])
def test_batch3_ragged_equals_three_single_runs(toy, wm):
    res3, cache3 = _decode(toy, PROMPTS, wm, 90)
    for b, p in enumerate(PROMPTS):
        (r1,), c1 = _decode(toy, [p], wm, 90)
        assert res3[b].tokens == r1.tokens, b
        if wm == "fp":  # fp16 draft weights: every kernel batch-invariant -> identical schedules
            assert res3[b].trace.to_ndjson() == r1.trace.to_ndjson(), b
        # a sequence that reached its budget first rode along (target-only rows) until the batch finished
        assert int(cache3.seq_lens()[b]) >= c1.seq_len
    # the short prompt (40 < 2G) exercised the short-fp1 top-up, the others the device flush
    assert any(s.flushed for s in res3[2].trace.steps) and any(s.flushed for s in res3[0].trace.steps)
    # ragged gamma_steps: some cycle ran a sequence below gamma (fp2 edge) while another drafted 4
    assert any(len(s.drafted) < 4 for r in res3 for s in r.trace.steps)


def test_batch_spec_equals_batch_ar_and_device_lengths(toy):
    res, cache = _decode(toy, PROMPTS, "int4", 70)
    logits, c2 = qs.prefill_batch(toy, PROMPTS, group_size=G, max_tokens=CAP)
    fw, _ = toy.device()
    ar = qs.ARAutoEngine(fw, c2)
    ar.set_pending([int(np.argmax(l)) for l in logits])
    toks = [[int(np.argmax(l))] for l in logits]
    for _ in range(69):
        out = ar.step()
        for b in range(3):
            toks[b].append(int(out[b]))
    for b in range(3):
        assert res[b].tokens[:70] == toks[b][:70], b
    # device lengths == host mirror, per sequence
    nb = cache.d_n_blocks.cpu().numpy()
    assert np.array_equal(nb * G, cache._nq)
    assert np.array_equal(cache.d_fp1_len.cpu().numpy(), cache._fp1)
    assert np.array_equal(cache.d_fp2_len.cpu().numpy(), cache._fp2[:, 0])
    assert np.array_equal(cache.d_pos.cpu().numpy(), cache.seq_lens())


def test_batch_state_machine_matches_oracle(toy):
    """Drive the oracle cache of each sequence with the accept sequence the device produced:
    quantised count, fp1 and fp2 lengths agree after every cycle's flush."""
    res, cache = _decode(toy, PROMPTS, "fp", 80)
    for b, p in enumerate(PROMPTS):
        oc = O.OracleKVCache(O.Layout(TOY.num_layers, TOY.num_heads, TOY.head_dim, G))
        n_quant = ((len(p) - G) // G) * G if len(p) >= G else 0
        fp1 = min(G, len(p) - n_quant)
        oc.quantized_token_count, oc.fp1_len = n_quant, fp1
        oc.fp2_lens[:] = len(p) - n_quant - fp1
        n_emitted = 1
        for s in res[b].trace.steps:
            g = len(s.drafted)
            assert g == max(0, min(4, oc.fp2_space() - 1, 80 - n_emitted))  # Q/specdec.py:329-333
            oc.fp2_lens += s.accepted + 1
            assert bool(oc.flush_if_full()) == s.flushed
            n_emitted += len(s.emitted)
        # tokens past the budget were still decoded for the batch, so compare up to the last record
        assert oc.quantized_token_count <= int(cache._nq[b])


def _rank_worker(rank, world, port, out):
    """One process per rank (both on cuda:0 here, one GPU each under torchrun): its partition of the
    job's sequences in one ragged-batch engine, job accounting over the process group (bench.py)."""
    import os

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_10424_b200.parallel import job_throughput, partition

        w = qs.init_weights(TOY, seed=7)
        mine = list(partition(len(JOB), world, rank))
        res, _ = _decode(w, [JOB[i] for i in mine], "int4", 30)
        jt = job_throughput(sum(len(r.tokens) for r in res), 1.0 + rank)
        out[rank] = (mine, [r.tokens for r in res], jt.total_units, jt.max_seconds)
    finally:
        dist.destroy_process_group()


JOB = [np.random.default_rng(s).integers(0, 64, size=n) for s, n in ((41, 200), (42, 251), (43, 90), (44, 333), (45, 140))]


def test_batch_partition_over_two_ranks_equals_one_batch(toy):
    """Config 4's batch partition: 5 sequences over 2 ranks (3 + 2, each rank its own engine) emit
    exactly the tokens of one 5-sequence batch, and the job accounting sums tokens / maxes time."""
    import socket

    import torch.multiprocessing as mp

    ref, _ = _decode(toy, JOB, "int4", 30)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = mp.Manager().dict()
    mp.spawn(_rank_worker, args=(2, port, out), nprocs=2, join=True)
    got = {}
    for r in range(2):
        mine, toks, total, mx = out[r]
        assert total == sum(len(x.tokens) for x in ref) and mx == 2.0
        got.update(dict(zip(mine, toks)))
    assert [got[i] for i in range(len(JOB))] == [r.tokens for r in ref]
