"""ZVE stage 2 on the GPU (espo_reshape_rewards): bit-exact against the oracle's
reshape_reward (fp64 arithmetic, f32 results), then through espo_prepare."""
import numpy as np
import pytest
import torch

from oracle import espo_oracle as O
from paper_2512_07710_b200.espo import Espo
from tests.gpu_common import require_cuda, to_dev

pytestmark = pytest.mark.gpu


def responses(seed, R, max_len):
    rng = np.random.default_rng(seed)
    seqs = []
    for i in range(R):
        n = int(rng.integers(0, max_len + max_len // 4))
        kind = i % 4
        if kind == 0:                                    # fresh tokens
            s = rng.integers(0, 50000, size=n)
        elif kind == 1:                                  # looping tail
            per = int(rng.integers(1, 9))
            motif = rng.integers(0, 100, size=per)
            s = np.concatenate([rng.integers(0, 50000, size=n // 2),
                                np.resize(motif, n - n // 2)])
        elif kind == 2:                                  # small alphabet
            s = rng.integers(0, 3, size=n)
        else:                                            # repeated paragraphs
            para = rng.integers(0, 1000, size=max(1, n // 3))
            s = np.resize(para, n)
        seqs.append(s.astype(np.int32))
    return seqs


@pytest.mark.parametrize("ngram,gamma,thresh", [(4, 1.0, 0.2), (3, 0.5, 0.05), (1, 2.0, 0.5)])
def test_reshape_rewards_bit_exact(ngram, gamma, thresh):
    dev = require_cuda()
    max_len = 300
    seqs = responses(ngram, 64, max_len)
    so = np.zeros(len(seqs) + 1, np.int64)
    np.cumsum([len(s) for s in seqs], out=so[1:])
    toks = np.concatenate(seqs) if so[-1] else np.zeros(0, np.int32)
    base = (np.random.default_rng(3).uniform(size=len(seqs)) < 0.5).astype(np.float32)
    ctx = Espo(1000, device=dev.index)
    out, lpen, rpen = ctx.reshape_rewards(to_dev(base, torch.float32, dev),
                                          to_dev(toks, torch.int32, dev),
                                          to_dev(so, torch.int64, dev), int(so[-1]), max_len,
                                          ngram=ngram, gamma_rep=gamma, rep_thresh=thresh)
    ctx.get_error()
    g32, t32 = float(np.float32(gamma)), float(np.float32(thresh))
    want = [O.reshape_reward(float(base[i]), seqs[i], max_len, ngram=ngram, gamma_rep=g32,
                             rep_thresh=t32) for i in range(len(seqs))]
    assert np.array_equal(out.cpu().numpy(), np.array([w[0] for w in want], np.float32))
    assert np.array_equal(lpen.cpu().numpy(), np.array([w[1] for w in want], np.float32))
    assert np.array_equal(rpen.cpu().numpy(), np.array([w[2] for w in want], np.float32))
    assert (rpen.cpu().numpy() < 0).any() and (lpen.cpu().numpy() < 0).any()
    ctx.close()


def test_reshaping_feeds_prepare():
    """An all-correct group of different lengths is zero-variance before reshaping and not
    after, on the GPU path end to end."""
    dev = require_cuda()
    lengths = [30, 60, 95, 120, 40, 40, 40, 40]          # group 0 varied, group 1 equal
    seqs = [np.arange(n, dtype=np.int32) for n in lengths]
    so = np.zeros(9, np.int64)
    np.cumsum(lengths, out=so[1:])
    toks = np.concatenate(seqs)
    base = np.ones(8, np.float32)
    gid = np.repeat(np.arange(2, dtype=np.int32), 4)
    ctx = Espo(1000, device=dev.index)
    shaped, _, _ = ctx.reshape_rewards(to_dev(base, torch.float32, dev),
                                       to_dev(toks, torch.int32, dev), to_dev(so, torch.int64, dev),
                                       int(so[-1]), 100)
    zv = torch.empty(8, dtype=torch.uint8, device=dev)
    ctx.prepare(shaped, to_dev(gid, torch.int32, dev), to_dev(so, torch.int64, dev),
                n_tokens=int(so[-1]), zv_out=zv)
    ctx.get_error()
    assert zv.cpu().numpy().tolist() == [0] * 4 + [1] * 4
    ctx.close()
