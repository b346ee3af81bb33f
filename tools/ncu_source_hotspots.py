"""Top CUDA source lines of an ncu report by warp-stall samples (needs -lineinfo and
--import-source on at capture time).

Usage: python tools/ncu_source_hotspots.py gpurun_out/prof.ncu-rep [--top 15] [--json out.json]
       (or the `ncu -i REP --page source --csv --print-source sass,cuda` export, .csv or .csv.gz)
Reports each source line's share of all stall samples, and the share on the RK4 loop body
(the lines of integrate<>, identified by their k1..k4 / a,b,c / s-update statements).
"""
import argparse
import csv
import io
import json
import re
import subprocess

# the RK4 loop body and the inlined FP64 helpers it is made of (dadd/dsub/dmul are also used a few
# times per character, so this share is an upper bound on the loop's share)
RK4_LINE = re.compile(r"\bk[1-4][xyz]\b|\b[abc][xyz] = |\bs[xyz] = |dmul\(h6|__fma_rn\(h6|"
                      r"for \(uint32_t it = 0; it < C\.n_it|return __d(add|sub|mul)_rn")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=15)
    ap.add_argument("--json")
    a = ap.parse_args()
    if a.rep.endswith((".csv", ".csv.gz")):  # the source page exported on the box (rep too big to ship)
        import gzip
        txt = (gzip.open if a.rep.endswith(".gz") else open)(a.rep, "rt").read()
    else:
        txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    out, file = [], ""
    samp_i = None
    for r in rows:
        if r and r[0] == "File Path":
            file = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            samp_i = r.index("Warp Stall Sampling (All Samples)")
        elif samp_i is not None and r and r[0].isdigit() and len(r) > samp_i:
            try:
                s = float(r[samp_i].replace(",", ""))
            except ValueError:
                continue
            if s > 0:
                out.append((s, f"{file}:{r[0]}", r[1].strip()))
    tot = sum(s for s, _, _ in out) or 1.0
    out.sort(reverse=True)
    rk4 = sum(s for s, _, t in out if RK4_LINE.search(t))
    res = {"report": a.rep, "total_samples": tot, "rk4_loop_share": round(rk4 / tot, 4),
           "top": [{"line": ln, "share": round(s / tot, 4), "source": t[:110]} for s, ln, t in out[:a.top]]}
    print(json.dumps(res, indent=1))
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
