"""Turn the raw ncu outputs of a round (gpurun_out/) into the committed summaries under
profiles/<tag>/:  launches.md (per-kernel share of a step from the gpu__time_duration launch
list), ncu_<name>.md (key metrics of each `--set full` capture), traffic.md + the
profiles/ncu_traffic.json that bench.py reads for roofline.traffic (DRAM bytes per sweep
launch averaged over one step's launches)."""
import csv
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import launch_summary  # noqa: E402
import ncu_summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def full_capture_md(rep, title):
    hdr, units, rows = raw_rows(rep)
    lines = [f"# {title}", "", f"source: `{os.path.basename(rep)}` (ncu --set full "
             "--clock-control none --import-source on; cold-cache replays)", ""]
    for n, vals in enumerate(rows):
        lines.append(f"## launch {n}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for w in ncu_summary.WANT:
            for i, h in enumerate(hdr):
                if h == w:
                    lines.append(f"| `{w}` | {vals[i]} | {units[i]} |")
        lines.append("")
    return "\n".join(lines)


def traffic(csv_path):
    """Mean DRAM bytes per espo_loss_fwd / espo_loss_bwd call from a metrics launch list."""
    with open(csv_path) as f:
        lines = [l for l in f if l.startswith('"')]
    per = {}
    for r in csv.DictReader(lines):
        k = launch_summary.short(r["Kernel Name"])
        if not k.startswith("k_"):
            continue
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"].lower()
        scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(u, 1)
        per.setdefault((r["ID"], k), {})[r["Metric Name"]] = v * scale
    fwd, bwd = [], []
    for (i, k), m in per.items():
        b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        if k.startswith(("k_rowstats", "k_fwd_rows")):
            fwd.append((int(i), k, b, m.get("gpu__time_duration.sum", 0)))
        if k.startswith(("k_dlogits", "k_bwd_rows", "k_bwd_recs")):
            bwd.append((int(i), k, b, m.get("gpu__time_duration.sum", 0)))
    nf = len([x for x in fwd if x[1].startswith("k_rowstats")])
    nb = len([x for x in bwd if x[1].startswith("k_dlogits")])
    return {"fwd_bytes_per_launch": sum(x[2] for x in fwd) / max(nf, 1),
            "bwd_bytes_per_launch": sum(x[2] for x in bwd) / max(nb, 1),
            "fwd_launches": nf, "bwd_launches": nb,
            "fwd_ms_total": sum(x[3] for x in fwd) / 1e6, "bwd_ms_total": sum(x[3] for x in bwd) / 1e6}


def main(tag, out_dir="gpurun_out"):
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    src = os.path.join(ROOT, out_dir)
    ll = os.path.join(src, "launches.csv")
    if os.path.exists(ll):
        shutil.copy(ll, os.path.join(dst, "launches.csv"))
        import io
        import contextlib
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            launch_summary.main(ll)
        open(os.path.join(dst, "launches.md"), "w").write(
            "# ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n"
            "Command: `python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg` "
            "(cold-cache serialised per-launch times: compare shares, not absolutes).\n\n"
            + buf.getvalue())
    for name in ("fwd", "bwd"):
        rep = os.path.join(src, f"prof_{name}.ncu-rep")
        if os.path.exists(rep):
            open(os.path.join(dst, f"ncu_{name}.md"), "w").write(
                full_capture_md(rep, f"K{'2' if name == 'fwd' else '5'} {name} sweep"))
    tr = os.path.join(src, "traffic.csv")
    if os.path.exists(tr):
        t = traffic(tr)
        t["source"] = f"profiles/{tag}/traffic.csv (ncu dram__bytes_read/write over one step)"
        jp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(jp):    # keep the factored-mode entries (written from their own capture)
            old = json.load(open(jp))
            t.update({k: v for k, v in old.items() if k.startswith("factored")})
        shutil.copy(tr, os.path.join(dst, "traffic.csv"))
        json.dump(t, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
        open(os.path.join(dst, "traffic.md"), "w").write(
            "# DRAM traffic per sweep launch (one step, ncu)\n\n```\n" + json.dumps(t, indent=1)
            + "\n```\n")
    fl = os.path.join(src, "launches_factored.csv")
    if os.path.exists(fl):      # factored-gradient mode: launch shares + DRAM bytes per sweep
        shutil.copy(fl, os.path.join(dst, "launches_factored.csv"))
        import io
        import contextlib
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            launch_summary.main(fl)
        open(os.path.join(dst, "launches_factored.md"), "w").write(
            "# ncu launch list, factored-gradient mode (gpu__time_duration.sum, --clock-control none)\n\n"
            "Command: `python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --factored` "
            "(cold-cache serialised per-launch times: compare shares, not absolutes).\n\n"
            + buf.getvalue())
        with open(fl) as f:
            lines = [l for l in f if l.startswith('"')]
        per = {}
        for r in csv.DictReader(lines):
            if "k_fwd_grad" not in r["Kernel Name"]:
                continue
            u = r["Metric Unit"].lower()
            sc = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1, "usecond": 1e3,
                  "msecond": 1e6}.get(u, 1)
            per.setdefault(int(r["ID"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * sc
        ids = sorted(per)
        jp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        t = json.load(open(jp)) if os.path.exists(jp) else {}
        n_step = int(t.get("bwd_launches") or 64)     # calls per step of the default chunking
        last = ids[-n_step:] if len(ids) >= n_step else ids
        t["factored_bytes_per_launch"] = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in last) / max(len(last), 1)
        t["factored_launches"] = len(last)
        t["factored_ms_total"] = sum(per[i].get("gpu__time_duration.sum", 0) for i in last) / 1e6
        t["factored_source"] = f"profiles/{tag}/launches_factored.csv (ncu dram__bytes_read/write of k_fwd_grad* over the last step of bench.py --factored --steps 1)"
        json.dump(t, open(jp, "w"), indent=1)
    rep = os.path.join(src, "prof_factored.ncu-rep")
    if os.path.exists(rep):
        open(os.path.join(dst, "ncu_factored.md"), "w").write(
            full_capture_md(rep, "k_fwd_grad_ring (factored-gradient sweep, default geometry)"))
    for name, title in (("tp8", "K2 on 1/8-vocabulary shard rows (TP8 emulation, 8192-row chunk)"),
                        ("gemm", "tcgen05 GEMMs of the LM-head backward (dh, dW), d = 4096, 8192-row sub-chunk"),
                        ("lmdz", "k_lmhead_dz (LM-head backward recompute + dz epilogue), d = 4096")):
        rep = os.path.join(src, f"prof_{name}.ncu-rep")
        if os.path.exists(rep):
            open(os.path.join(dst, f"ncu_{name}.md"), "w").write(full_capture_md(rep, title))
    for ll_name, title in (("launches_lmhead_bwd", "LM-head backward, d = 4096, 8192 rows: per-launch "
                            "time and DRAM bytes (ncu --cache-control none --clock-control none)"),
                           ("launches_lmhead_bwd_cublas", "same, dh/dW on cuBLAS (A/B option)")):
        lp = os.path.join(src, ll_name + ".csv")
        if os.path.exists(lp):
            import io
            import contextlib
            sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
            import launch_table
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                launch_table.main(lp, 20.0)
            shutil.copy(lp, os.path.join(dst, ll_name + ".csv"))
            open(os.path.join(dst, ll_name + ".md"), "w").write(
                f"# {title}\n\n```\n" + buf.getvalue() + "```\n")
    for f in ("bench_full.json", "bench_full.err", "gpu_tests.log", "smoke.log", "bench_tp8.json",
              "bench_C4_strong_verify.json", "bench_C1_strong_verify.json",
              "bench_C1_emulate2.json", "bench_C1_emulate4.json", "bench_C1_emulate8.json",
              "bench_C4_emulate8.json", "bench_lmhead_bwd_dense.json",
              "bench_lmhead_fwd_d4096.json", "bench_lmhead_fwd_d8192.json",
              "ncu_lmhead_fwd_d4096.csv", "ncu_lmhead_fwd_d8192.csv",
              "bench_lmhead_bwd_realistic.json", "gemm_sweep.json"):
        p = os.path.join(src, f)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(dst, f))
    print("wrote", dst)


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
