"""Full-size parity at BASELINE.json sizes, in the launch configuration bench.py times
(32,768-row chunks, default kernel variants, bf16 logits and gradients).

C1 (64 × 8 × 4096, V = 151,936): every token's statistics, decisions, counts and the global
loss against the full oracle; dlogits on rows sampled from several bwd chunks.
C3 (256 × 16 × ≤8192, 60 % zero-variance groups, lognormal lengths, chunks splitting
sequences): per-rollout results on sampled prompt groups against the oracle run on those
groups, and size-independent properties (loss = −ΣJ_i/N, exact counts) for the whole batch.

Logits: 1024 distinct rows (espo_synth recipe) tiled over the chunk buffer; batch row t reads
distinct row t mod 1024, so the oracle evaluates O2 once per (row, token) pair.
"""
import numpy as np
import pytest
import torch

import espo_synth as S
from oracle import espo_oracle as O
from tests.gpu_common import (check_dlogits_bf16, decision_aware_reference, oracle_cfg,
                              require_cuda, to_dev)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
U_ROWS = 1024
CHUNK = 32768


class Cycled:
    def __init__(self, rows):
        self.rows = rows

    def __getitem__(self, t):
        return self.rows[t % self.rows.shape[0]]


class Batch:
    pass


def build(name, dev, seed=None):
    w = S.WORKLOADS[name]
    seed = S.config_seed(w.index) if seed is None else seed
    b = Batch()
    b.w, b.V = w, w.V
    b.group_ids, b.seq_offsets = S.make_layout(w, seed)
    b.rewards = S.make_rewards(w, seed)
    b.T = int(b.seq_offsets[-1])
    rows = S.make_logit_rows(U_ROWS, w.V, seed, dtype="bf16")
    tok_u = S.sample_tokens_gumbel(rows, seed)
    lp_u = np.array([O.row_stats(rows[r], int(tok_u[r]))[1] for r in range(U_ROWS)])
    idx = np.arange(b.T) % U_ROWS
    b.rows, b.tok_u = rows, tok_u
    b.tokens = tok_u[idx].astype(np.int32)
    b.old = S.drift_old_logp(lp_u[idx], b.seq_offsets, seed)
    b.logits = Cycled(rows)
    buf = torch.from_numpy(rows).to(dev).to(torch.bfloat16)
    # [CHUNK + 1024, V]: buffer row r = distinct r % 1024 (the extra 1024 rows let a chunk
    # starting at any batch row t0 use the view buf[t0 % 1024:])
    b.buf = buf.repeat(CHUNK // U_ROWS + 1, 1)
    return b


def run(b, dev, bwd_rows=None, cfgkw=None, factored=False):
    """prepare → fwd chunks → finalize → bwd chunks (32,768 rows, as bench.py). Returns the
    loss/stats and, for each (chunk_start, rows-in-chunk) in bwd_rows, the gradient rows.
    factored: espo_loss_fwd_factored chunks (G into one reused buffer, as bench.py --factored)
    and the gradient rows as espo_loss_row_scale · G in fp64."""
    from paper_2512_07710_b200.espo import Espo, stats_to_dict
    ctx = Espo(b.V, logits_dtype=torch.bfloat16, device=dev.index, **(cfgkw or {}))
    tok = to_dev(b.tokens, torch.int32, dev)
    old = to_dev(b.old, torch.float32, dev)
    ctx.prepare(to_dev(b.rewards, torch.float32, dev), to_dev(b.group_ids, torch.int32, dev),
                to_dev(b.seq_offsets, torch.int64, dev), n_tokens=b.T)
    if factored:
        dl = torch.empty((CHUNK, b.V), dtype=torch.bfloat16, device=dev)
        Gs = {}
        for c0 in range(0, b.T, CHUNK):
            c1 = min(b.T, c0 + CHUNK)
            ctx.loss_fwd_factored(b.buf[:c1 - c0], tok[c0:c1], old[c0:c1], None, grad=dl[:c1 - c0],
                                  row_begin=c0)
            if bwd_rows and c0 in bwd_rows:
                Gs[c0] = dl[torch.as_tensor(bwd_rows[c0], device=dev)].double().cpu().numpy()
        loss, stats = ctx.loss_finalize()
        scale = ctx.loss_row_scale().double().cpu().numpy()
        ctx.get_error()
        grads = {c0: scale[c0 + np.asarray(bwd_rows[c0])][:, None] * G for c0, G in Gs.items()}
        return ctx, float(loss.item()), stats_to_dict(stats), grads
    for c0 in range(0, b.T, CHUNK):
        c1 = min(b.T, c0 + CHUNK)
        ctx.loss_fwd(b.buf[:c1 - c0], tok[c0:c1], old[c0:c1], None, row_begin=c0)
    loss, stats = ctx.loss_finalize()
    grads = {}
    dl = torch.empty((CHUNK, b.V), dtype=torch.bfloat16, device=dev)
    for c0 in range(0, b.T, CHUNK):
        c1 = min(b.T, c0 + CHUNK)
        ctx.loss_bwd(b.buf[:c1 - c0], dl[:c1 - c0], row_begin=c0)
        if bwd_rows and c0 in bwd_rows:
            sel = torch.as_tensor(bwd_rows[c0], device=dev)
            grads[c0] = dl[sel].float().cpu().numpy()
    ctx.get_error()
    return ctx, float(loss.item()), stats_to_dict(stats), grads


@pytest.mark.parametrize("factored", [False, True], ids=["two_sweep", "factored"])
def test_c1_full_size(factored):
    dev = require_cuda()
    b = build("C1", dev)
    rng = np.random.default_rng(0)
    chunks = [0, 5 * CHUNK, b.T - CHUNK]
    bwd_rows = {c: np.sort(rng.choice(CHUNK, 48, replace=False)) for c in chunks}
    ctx, loss, st, grads = run(b, dev, bwd_rows, factored=factored)
    tok = {k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()}
    rol = {k: v.cpu().numpy() for k, v in ctx.export_rollout_stats().items()}
    ctx.close()

    cfg = oracle_cfg(b.V)
    memo = {}
    ref = O.espo_loss(b.logits, b.tokens, b.old, None, b.rewards, b.group_ids, b.seq_offsets,
                      cfg, row_key=lambda t: t % U_ROWS, stats_cache=memo)
    # exact fields
    assert np.array_equal(rol["zv"].astype(bool), ref.zv)
    assert np.array_equal(rol["active"].astype(bool), ref.active)
    assert np.array_equal(rol["adv"], ref.adv)
    for k in ("n_active_rollouts", "n_active_tokens", "n_zv_groups", "n_groups"):
        assert st[k] == ref.stats[k], k
    v = ref.kappa >= 0
    assert np.array_equal(tok["valid"].astype(bool), v)
    for name, tol in (("lse", 2e-6), ("lp", 2e-6), ("H", 1e-5)):
        want = getattr(ref, name)[v]
        got = tok[name][v].astype(np.float64)
        d = np.abs(got - want) / (tol * np.maximum(1, np.abs(want)))
        w = np.argsort(d)[-5:]
        assert np.all(d <= 1), (name, d.max(), got[w], want[w], ref.lp[v][w], ref.H[v][w])
    dq = np.abs(tok["q"][v].astype(np.float64) - ref.q[v])
    assert np.all(dq <= 1e-5 * ref.q[v] + 1e-30)

    class Inst:   # decision-aware protocol needs .seq_offsets and .run
        seq_offsets = b.seq_offsets

        @staticmethod
        def run(c, **kw):
            return O.espo_loss(b.logits, b.tokens, b.old, None, b.rewards, b.group_ids,
                               b.seq_offsets, c, row_key=lambda t: t % U_ROWS,
                               stats_cache=memo, **kw)

    g = {"tok": tok}
    ref2, flips = decision_aware_reference(g, Inst, ref, cfg)
    floor = float(np.abs(ref2.J_i).sum()) / ref2.denom
    assert abs(loss - ref2.loss) <= 1e-5 * (abs(ref2.loss) + floor), (loss, ref2.loss)
    # coefficients c_t (= ∂J_i/∂lp_t before 1/N) for every active token
    dc = np.abs(tok["coef"][v].astype(np.float64) - ref2.coef[v])
    assert np.all(dc <= 1e-5 * np.abs(ref2.coef[v]) + 1e-12)
    # gradient rows sampled from three bwd chunks
    for c0, rows in bwd_rows.items():
        want = np.stack([O.dlogits_row(ref2, c0 + r, b.logits[c0 + r], int(b.tokens[c0 + r]), cfg)
                         for r in rows])
        check_dlogits_bf16(grads[c0], want)


@pytest.mark.parametrize("name", ["C3", "C2", "C4"])
def test_full_size_sampled_groups(name):
    """C3 (variable lengths, 60 % eliminated groups, chunks splitting sequences), C2
    (32 × 16 × 32,768 long-CoT sequences, each spanning a whole 32,768-row chunk) and C4
    (512 × 16 × 16,384 = 134 M tokens: the largest configuration, on one GPU)."""
    dev = require_cuda()
    b = build(name, dev)
    ctx, loss, st, _ = run(b, dev)
    rol = {k: v.cpu().numpy() for k, v in ctx.export_rollout_stats().items()}
    G = b.w.G
    zv_groups = int(rol["zv"].reshape(-1, G)[:, 0].sum())
    assert zv_groups == st["n_zv_groups"]
    if b.w.forced_zv:
        assert zv_groups == b.w.forced_zv
    assert st["n_groups"] == b.w.n_prompts
    N = int(rol["active"].sum())
    assert st["n_active_rollouts"] == N
    # property at any size: loss = −ΣJ_i / N (fp64 sums on both sides)
    assert loss == pytest.approx(-rol["J"].sum() / N, rel=1e-6)
    T_act = int(np.diff(b.seq_offsets)[rol["active"].astype(bool)].sum())
    assert st["n_active_tokens"] == T_act     # no masking in C2/C3
    # sampled groups: two active, one eliminated, rerun by the oracle on their own
    active_groups = [g for g in range(b.w.n_prompts) if not rol["zv"][g * G]]
    zv_g = [g for g in range(b.w.n_prompts) if rol["zv"][g * G]]
    cfg = oracle_cfg(b.V)
    picks = [active_groups[0], active_groups[len(active_groups) // 2]] + zv_g[:1]
    if name in ("C2", "C4"):
        picks = picks[:1] + zv_g[:1]     # one 16 × 32k group is 524k tokens for the oracle
    for g in picks:
        r0, r1 = g * G, (g + 1) * G
        t0, t1 = int(b.seq_offsets[r0]), int(b.seq_offsets[r1])
        so = b.seq_offsets[r0:r1 + 1] - t0
        memo = {}
        key = (lambda u, t0=t0: (u + t0) % U_ROWS)   # distinct row of local row u
        sub = O.espo_loss(Cycled(np.roll(b.rows, -(t0 % U_ROWS), axis=0)), b.tokens[t0:t1],
                          b.old[t0:t1], None, b.rewards[r0:r1], b.group_ids[r0:r1], so, cfg,
                          row_key=key, stats_cache=memo)
        assert np.array_equal(rol["adv"][r0:r1], sub.adv)
        assert np.array_equal(rol["active"][r0:r1].astype(bool), sub.active)
        tok = {k: v.cpu().numpy() for k, v in ctx.export_token_stats(t0, t1 - t0).items()}
        v = sub.kappa >= 0
        assert np.array_equal(tok["valid"].astype(bool), v)
        if not v.any():
            continue
        assert np.allclose(tok["lp"][v], sub.lp[v], rtol=0, atol=2e-6 * max(1, np.abs(sub.lp[v]).max()))
        gb, gc = tok["bucket"].astype(np.int64), tok["clip"].astype(np.int64)
        if np.array_equal(gb[v], sub.bucket[v]) and np.array_equal(gc[v], 1 - sub.kappa[v]):
            np.testing.assert_allclose(rol["J"][r0:r1], sub.J_i, rtol=1e-5,
                                       atol=1e-5 * np.abs(sub.J_i).max())
            dc = np.abs(tok["coef"][v].astype(np.float64) - sub.coef[v])
            assert np.all(dc <= 1e-5 * np.abs(sub.coef[v]) + 1e-12)
        else:   # a flip within rounding: decisions must sit at the oracle's kinks
            class Inst:
                seq_offsets = so

                @staticmethod
                def run(c, **kw):
                    return O.espo_loss(Cycled(np.roll(b.rows, -(t0 % U_ROWS), axis=0)),
                                       b.tokens[t0:t1], b.old[t0:t1], None, b.rewards[r0:r1],
                                       b.group_ids[r0:r1], so, c, row_key=key,
                                       stats_cache=memo, **kw)
            sub2, _ = decision_aware_reference({"tok": tok}, Inst, sub, cfg)
            np.testing.assert_allclose(rol["J"][r0:r1], sub2.J_i, rtol=1e-5,
                                       atol=1e-5 * np.abs(sub2.J_i).max())
    ctx.close()


def _rollout_chunks(so, max_rows):
    chunks, s = [], 0
    for i in range(1, len(so)):
        if so[i] - s > max_rows:
            chunks.append((s, int(so[i - 1])))
            s = int(so[i - 1])
    if so[-1] > s:
        chunks.append((s, int(so[-1])))
    return chunks


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_full_size_single_pass_is_bitwise_two_sweep(name):
    """At full size in the bench launch configuration, the single-pass mode (espo_set_mask +
    espo_loss_fwd_bwd on chunks of whole rollouts) reproduces the two-sweep pass bit for bit:
    loss, statistics and sampled gradient rows from every chunk."""
    from paper_2512_07710_b200.espo import Espo, stats_to_dict
    dev = require_cuda()
    b = build(name, dev)
    rng = np.random.default_rng(1)
    tok = to_dev(b.tokens, torch.int32, dev)
    old = to_dev(b.old, torch.float32, dev)
    args = (to_dev(b.rewards, torch.float32, dev), to_dev(b.group_ids, torch.int32, dev),
            to_dev(b.seq_offsets, torch.int64, dev))
    dl = torch.empty((CHUNK, b.V), dtype=torch.bfloat16, device=dev)

    def view(c0, c1):
        o = c0 % U_ROWS
        return b.buf[o:o + (c1 - c0)]

    def pick(c0, c1):
        return np.sort(rng.choice(c1 - c0, min(16, c1 - c0), replace=False))

    # two sweeps, chunks of CHUNK rows
    ctx = Espo(b.V, logits_dtype=torch.bfloat16, device=dev.index)
    ctx.prepare(*args, n_tokens=b.T)
    tiles = [(c0, min(b.T, c0 + CHUNK)) for c0 in range(0, b.T, CHUNK)]
    for c0, c1 in tiles:
        ctx.loss_fwd(view(c0, c1), tok[c0:c1], old[c0:c1], None, row_begin=c0)
    loss2, st2 = ctx.loss_finalize()
    ref_rows = {}
    single_chunks = _rollout_chunks(b.seq_offsets, CHUNK)
    want_rows = {c0: c0 + pick(c0, c1) for c0, c1 in single_chunks}
    flat = np.concatenate(list(want_rows.values()))
    for c0, c1 in tiles:
        ctx.loss_bwd(view(c0, c1), dl[:c1 - c0], row_begin=c0)
        sel = flat[(flat >= c0) & (flat < c1)]
        if len(sel):
            got = dl[torch.as_tensor(sel - c0, device=dev)].cpu()
            for k, t in enumerate(sel):
                ref_rows[int(t)] = got[k]
    ctx.get_error()
    loss2, st2 = float(loss2.item()), stats_to_dict(st2)
    ctx.close()
    # single pass, chunks of whole rollouts
    ctx = Espo(b.V, logits_dtype=torch.bfloat16, device=dev.index)
    ctx.prepare(*args, n_tokens=b.T)
    ctx.set_mask(None)
    for c0, c1 in single_chunks:
        ctx.loss_fwd_bwd(view(c0, c1), tok[c0:c1], old[c0:c1], dl[:c1 - c0], row_begin=c0)
        sel = want_rows[c0]
        got = dl[torch.as_tensor(sel - c0, device=dev)].cpu()
        for k, t in enumerate(sel):
            assert torch.equal(got[k], ref_rows[int(t)]), (c0, int(t))
    loss1, st1 = ctx.loss_finalize()
    ctx.get_error()
    ctx.close()
    assert float(loss1.item()) == loss2
    assert stats_to_dict(st1) == st2


def test_c3_full_size_rlzvp():
    """C3 at full size with RL-ZVP (ZVE stage 3): the 154 uniform-reward groups are read and
    get entropy-shaped token advantages instead of being eliminated. Exact counts, loss =
    −ΣJ_i/N, and one zero-variance and one mixed group against the oracle (the RL-ZVP token
    advantage is a difference of fp32 entropies: absolute tolerance β·4e-5)."""
    dev = require_cuda()
    b = build("C3", dev)
    ctx, loss, st, _ = run(b, dev, cfgkw={"zv_mode": O.ZV_RLZVP})
    rol = {k: v.cpu().numpy() for k, v in ctx.export_rollout_stats().items()}
    G = b.w.G
    assert st["n_zv_groups"] == b.w.forced_zv
    assert st["n_active_rollouts"] == int((np.diff(b.seq_offsets) > 0).sum())
    assert st["n_active_tokens"] == b.T
    N = int(rol["active"].sum())
    assert loss == pytest.approx(-rol["J"].sum() / N, rel=1e-6)
    cfg = oracle_cfg(b.V, zv_mode=O.ZV_RLZVP)
    zv_g = [g for g in range(b.w.n_prompts) if b.rewards[g * G:(g + 1) * G].min() ==
            b.rewards[g * G:(g + 1) * G].max()]
    mixed = [g for g in range(b.w.n_prompts) if g not in set(zv_g)]
    compared = 0
    for g in (zv_g[0], zv_g[len(zv_g) // 2], zv_g[-1], mixed[0], mixed[-1]):
        r0, r1 = g * G, (g + 1) * G
        t0, t1 = int(b.seq_offsets[r0]), int(b.seq_offsets[r1])
        so = b.seq_offsets[r0:r1 + 1] - t0
        key = (lambda u, t0=t0: (u + t0) % U_ROWS)
        sub = O.espo_loss(Cycled(np.roll(b.rows, -(t0 % U_ROWS), axis=0)), b.tokens[t0:t1],
                          b.old[t0:t1], None, b.rewards[r0:r1], b.group_ids[r0:r1], so, cfg,
                          row_key=key, stats_cache={})
        tok = {k: v.cpu().numpy() for k, v in ctx.export_token_stats(t0, t1 - t0).items()}
        v = sub.kappa >= 0
        assert np.array_equal(tok["valid"].astype(bool), v) and v.all()
        gb, gc = tok["bucket"].astype(np.int64), tok["clip"].astype(np.int64)
        if not (np.array_equal(gb, sub.bucket) and np.array_equal(gc, 1 - sub.kappa)):
            continue          # a decision at a kink (checked elsewhere); values not comparable
        atol = cfg.zvp_beta * 4e-5 if g in zv_g else 0.0
        np.testing.assert_allclose(rol["J"][r0:r1], sub.J_i, rtol=1e-5,
                                   atol=atol + 1e-5 * np.abs(sub.J_i).max() * (g not in zv_g))
        compared += 1
    assert compared >= 3
    ctx.close()
