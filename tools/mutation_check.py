"""Mutation check for the oracle's pins (TEST TOOLING; runs on CPU, touches only a scratch copy).

Each mutation is a plausible mistake in oracle/espo_oracle.py. For each one this copies
oracle/, tests/ and espo_synth/ into a temporary directory, applies the mutation, and runs
the oracle pins (`pytest -m "not gpu" tests/test_oracle_*.py -x`). A mutation that passes
every pin is a gap in the pins. Exit code 0 iff every mutation is caught.

    python tools/mutation_check.py            # all mutations
    python tools/mutation_check.py -k eps     # those whose name contains "eps"
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, old text, new text) applied to oracle/espo_oracle.py
MUTATIONS = [
    ("supplied_entropies_ignored (reading Q4's alternative not wired)",
     "            H = np.asarray(entropy, dtype=np.float64)[valid]\n",
     "            pass\n"),
    ("eps_from_sequence_mean_entropy (Eq. 3 over the whole sequence, not per bucket)",
     "        s, eps = bucket_ratio_clip(lp[sel], old[sel], H[sel], cfg)\n",
     "        s, _ = bucket_ratio_clip(lp[sel], old[sel], H[sel], cfg)\n"
     "        _, eps = bucket_ratio_clip(lp, old, H, cfg)\n"),
    ("s_from_whole_sequence (GSPO ratio, Eq. 2 not per bucket)",
     "        s, eps = bucket_ratio_clip(lp[sel], old[sel], H[sel], cfg)\n",
     "        _, eps = bucket_ratio_clip(lp[sel], old[sel], H[sel], cfg)\n"
     "        s, _ = bucket_ratio_clip(lp, old, H, cfg)\n"),
    ("weight_1_over_n (instead of 1/(nb*|y_tau|))",
     "w = 1.0 / (nb * size) if", "w = 1.0 / n if"),
    ("weight_drops_1_over_nb",
     "w = 1.0 / (nb * size) if", "w = 1.0 / size if"),
    ("weight_drops_1_over_size",
     "w = 1.0 / (nb * size) if", "w = 1.0 / nb if"),
    ("clip_min_becomes_max",
     "ell = min(v * A, vc * A)", "ell = max(v * A, vc * A)"),
    ("kappa_wrong_direction",
     "kappa = not ((A > 0 and v > hi) or (A < 0 and v < lo))",
     "kappa = not ((A > 0 and v < lo) or (A < 0 and v > hi))"),
    ("dropped_logit_scale",
     "x = float(logit_scale) * np.asarray(z_row, dtype=np.float64)",
     "x = np.asarray(z_row, dtype=np.float64)"),
    ("split_rank_off_by_one",
     "return [max((cfg.split_num * n) // cfg.split_den, 1)]",
     "return [max((cfg.split_num * n) // cfg.split_den + 1, 1)]"),
    ("ties_to_high_bucket",
     "sum(1 for th in thetas if h > th)", "sum(1 for th in thetas if h >= th)"),
    ("entropy_sign_flip",
     "H = -float(np.sum(p[nz] * np.log(p[nz])))", "H = float(np.sum(p[nz] * np.log(p[nz])))"),
    ("eps_log2_instead_of_ln",
     "cfg.alpha * hsum / (n * math.log(cfg.vocab))", "cfg.alpha * hsum / (n * math.log2(cfg.vocab))"),
    ("eps_floor_dropped",
     "eps = max(cfg.eps_min, cfg.alpha", "eps = max(0.0, cfg.alpha"),
    ("s_sum_not_mean (geometric mean exponent 1/|y_tau| dropped)",
     "    m = delta / n\n", "    m = delta\n"),
    ("ratio_reading_R2_as_R1",
     "                v = s                     # sg[s_τ]·π_θ/sg[π_θ]: value s_τ\n",
     "                v = s * math.exp(lp[j] - old[j])\n"),
    ("advantage_unbiased_std_by_default",
     "denom = (n - 1) if cfg.std_unbiased else n", "denom = n if cfg.std_unbiased else (n - 1)"),
    ("advantage_eps_inside_sqrt",
     "(r[j] - mu) / (sigma + cfg.adv_eps)", "(r[j] - mu) / math.sqrt(var + cfg.adv_eps)"),
    ("zv_groups_not_eliminated",
     "        if grp[\"zv\"][i] and not zvp:\n            continue",
     "        if False:\n            continue"),
    ("normaliser_counts_all_rollouts",
     "denom = float(n_active if cfg.norm == NORM_SEQ else t_active)",
     "denom = float(R if cfg.norm == NORM_SEQ else t_active)"),
    ("dlogits_target_uses_minus_p",
     "dz[y] = lam * g * res.q[t]", "dz[y] = lam * g * (-p[y])"),
    ("dlogits_sign_flip",
     "g = -grad_loss * res.coef[t] / res.denom", "g = grad_loss * res.coef[t] / res.denom"),
]


def run_one(name, old, new, quiet=True):
    with tempfile.TemporaryDirectory(prefix="espo_mut_") as tmp:
        for d in ("oracle", "tests", "espo_synth"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__"))
        path = os.path.join(tmp, "oracle", "espo_oracle.py")
        src = open(path).read()
        if src.count(old) != 1:
            return name, "NOT APPLIED (pattern count %d)" % src.count(old)
        open(path, "w").write(src.replace(old, new))
        tests = sorted(f for f in os.listdir(os.path.join(tmp, "tests"))
                       if f.startswith("test_oracle_"))
        cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
               "-o", "addopts="] + [os.path.join("tests", t) for t in tests]
        r = subprocess.run(cmd, cwd=tmp, capture_output=True, text=True)
        if r.returncode == 0:
            return name, "SURVIVED"
        failed = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
        return name, "caught by " + (failed[0][7:].split(" - ")[0] if failed else f"rc={r.returncode}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="")
    args = ap.parse_args()
    bad = 0
    for name, old, new in MUTATIONS:
        if args.k and args.k not in name:
            continue
        name, verdict = run_one(name, old, new)
        print(f"{name:70s} {verdict}", flush=True)
        bad += not verdict.startswith("caught")
    print("all mutations caught" if bad == 0 else f"{bad} mutation(s) not caught")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
