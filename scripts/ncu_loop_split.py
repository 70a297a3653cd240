"""Split an ncu --set full report's warp-stall samples of one kernel into the
hot step loop (the most-executed instruction range) and the rest (tile
transitions), with the stall reasons and the top instructions outside the loop.

    python scripts/ncu_loop_split.py gpurun_out/prof_c3_it1.ncu-rep
"""
import csv
import io
import subprocess
import sys


def main(path, top=15):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    col = h.index
    isrc, iss, iex = col("Source"), col("Warp Stall Sampling (All Samples)"), col(
        "Instructions Executed")
    reasons = [c for c in h if c.startswith("stall_") and "(Not" not in c]
    ex = [int(r[iex] or 0) for r in data]
    mx = max(ex)
    loop = [i for i, e in enumerate(ex) if e > mx * 0.5]
    lo, hi = min(loop), max(loop)
    tot = sum(int(r[iss] or 0) for r in data)

    def agg(idx):
        s = {r: 0 for r in reasons}
        n = 0
        for i in idx:
            n += int(data[i][iss] or 0)
            for r in reasons:
                s[r] += int(data[i][col(r)] or 0)
        return n, {k: v for k, v in sorted(s.items(), key=lambda x: -x[1]) if v}

    n_in, s_in = agg(range(lo, hi + 1))
    n_out, s_out = agg([i for i in range(len(data)) if i < lo or i > hi])
    ins_in = sum(ex[lo:hi + 1])
    ins_out = sum(ex) - ins_in
    print(f"loop: SASS [{lo}, {hi}] ({hi - lo + 1} instructions); stall samples in loop "
          f"{n_in / tot:.3f}, outside {n_out / tot:.3f}; instructions executed outside "
          f"{ins_out / max(ins_in, 1):.3f} of the loop's")
    print("in loop:", s_in)
    print("outside:", s_out)
    outs = sorted(((int(data[i][iss] or 0), i, data[i][isrc].strip()) for i in range(len(data))
                   if i < lo or i > hi), reverse=True)[:top]
    for o in outs:
        print("  ", o)


if __name__ == "__main__":
    main(sys.argv[1])
