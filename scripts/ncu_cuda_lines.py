"""Per CUDA source line warp-stall samples from an
`ncu --page source --csv --print-source cuda,sass` export (the source-line
rows carry the line's aggregated metrics): the hottest lines with their
file, text and the largest stall reasons."""

import csv
import gzip
import sys


def main(path, top=40):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt", newline="")))
    cur_file, hdr, out = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0]:
            continue  # SASS rows
        d = dict(zip([f"{h}#{i}" for i, h in enumerate(hdr)], r))
        out.append((cur_file, r[0], r[1], r))
    i_all = hdr.index("Warp Stall Sampling (All Samples)")
    i_ni = hdr.index("Warp Stall Sampling (Not-issued Samples)")
    i_ex = hdr.index("Instructions Executed")
    stalls = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]

    def num(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    total = sum(num(r[i_all]) for _, _, _, r in out)
    out.sort(key=lambda t: -num(t[3][i_all]))
    print(f"total samples {total:.0f}")
    for f, ln, src, r in out[:top]:
        s = num(r[i_all])
        st = sorted(((num(r[i]), h[6:]) for i, h in stalls), reverse=True)[:3]
        sts = " ".join(f"{h}:{v:.0f}" for v, h in st if v > 0)
        print(f"{s:7.0f} {100 * s / total:5.1f}%  {f}:{ln:<5} ex {num(r[i_ex]):9.0f}  [{sts}]  {src.strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
