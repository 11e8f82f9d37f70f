"""Hottest lines of an `ncu --page source --csv --print-source sass` export:
per SASS instruction, the warp-stall samples (all / not issued), with its
address and text."""

import csv
import sys


def main(path, top=45):
    rows = list(csv.reader(open(path, newline="")))
    # the export may hold several files: each block starts with a header row
    hdr, recs, cur_file = None, [], None
    for r in rows:
        if not r:
            continue
        if r[0] in ("#", "Line", "Address", "Line No") or (len(r) > 1 and r[1] == "Source"):
            hdr = r
            continue
        if len(r) == 1 and r[0].startswith("File"):
            cur_file = r[0]
            continue
        if hdr is None or len(r) != len(hdr):
            if len(r) == 1:
                cur_file = r[0]
            continue
        recs.append((cur_file, dict(zip(hdr, r))))
    if not recs:
        print("no records; header:", hdr)
        return
    keys = list(recs[0][1].keys())
    samp = next((k for k in keys if "Warp Stall Sampling (All" in k), None)
    noiss = next((k for k in keys if "Warp Stall Sampling (Not" in k), None)
    print("columns:", [k for k in keys][:40])

    def num(x):
        try:
            return float(str(x).replace(",", ""))
        except ValueError:
            return 0.0
    recs.sort(key=lambda fr: -num(fr[1].get(samp, 0)))
    total = sum(num(fr[1].get(samp, 0)) for fr in recs)
    print(f"total samples {total:.0f}")
    for f, r in recs[:top]:
        s = num(r.get(samp, 0))
        src = (r.get("Source") or "").strip()[:110]
        print(f"{s:8.0f} {100 * s / max(total, 1):5.1f}%  ni {num(r.get(noiss, 0)):7.0f}  "
              f"{r.get('Address', r.get('#', '?'))}  {src}")


if __name__ == "__main__":
    main(sys.argv[1])
