"""Top source lines of an ncu report by warp-stall samples (`ncu -i rep --page source --csv`),
so a capture can be summarised on the GPU box and only a small table brought back.
usage: python tools/ncu_source_top.py report.ncu-rep [n] [samples|inst] [cuda|sass]"""
import csv
import io
import subprocess
import sys


def main(rep, n=40, key="samples", view="cuda"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        print("no source page")
        return
    hdr = rows[0]
    def col(*names):
        for nm in names:
            for i, h in enumerate(hdr):
                if h.strip().lower() == nm.lower():
                    return i
        return None
    i_line, i_src = col("#", "Line"), col("Source")
    i_samp = col("Warp Stall Sampling (All Samples)", "Sampling Data (All)")
    i_inst = col("Instructions Executed")
    data = []
    for r in rows[1:]:
        try:
            samp = float(r[i_samp]) if i_samp is not None and r[i_samp] else 0.0
            inst = float(r[i_inst]) if i_inst is not None and r[i_inst] else 0.0
        except ValueError:
            continue
        data.append((inst if key == "inst" else samp, r))
    tot = sum(x[0] for x in data) or 1.0
    print(f"columns: {hdr}")
    for samp, r in sorted(data, key=lambda x: -x[0])[:n]:
        line = r[i_line] if i_line is not None else "?"
        inst = r[i_inst] if i_inst is not None else ""
        src = (r[i_src] if i_src is not None else "").strip()[:110]
        print(f"{100 * samp / tot:6.2f}%  line {line:>5}  inst {inst:>12}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40,
         sys.argv[3] if len(sys.argv) > 3 else "samples", sys.argv[4] if len(sys.argv) > 4 else "cuda")
