"""Per-CTA timeline of the step kernel (measurement build, -DGS_TRACE=1).

    GS_NVCC_EXTRA=-DGS_TRACE=1 python -c "..._build to build/trace.so"
    python scripts/trace_k2.py --lib paper_2601_16736_b200/build/trace.so --rows 100000 --vis 0.5

Each CTA stamps %globaltimer at: 0 entry, 1 first chunk emitted (loader),
2 end marker emitted, 3 first chunk landed (consumer warp 0), 4 consumer
exit, 5 storer's writes complete, 6 block reduction done, 7 last-block
entry to the final reduction, 8 final reduction done, 11 exit; slot 9 =
visible rows of the CTA, 10 = SM id.  The cloud is stepped round robin with
others (L2-cold) and the traced launch is the last one.
"""

import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_16736_b200 import _lib as L  # noqa: E402
from paper_2601_16736_b200 import records as R  # noqa: E402
from paper_2601_16736_b200 import synthetic as S  # noqa: E402
from paper_2601_16736_b200.optimizer import AdamWGS  # noqa: E402

NAMES = {0: "entry", 1: "first emit", 2: "end emit", 3: "first chunk in", 4: "consumers out",
         5: "stores done", 6: "block reduce", 11: "exit"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", required=True)
    ap.add_argument("--rows", type=int, default=100_000)
    ap.add_argument("--vis", type=float, default=0.5)
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--clouds", type=int, default=6)
    args = ap.parse_args()
    lib = L.load(args.lib)
    L._lib = lib
    lib.gs_debug_set_trace.argtypes = [C.c_void_p]
    dev = torch.device("cuda:0")
    cfg = S.WorkloadConfig(n=args.rows, p_vis=args.vis, seed=3)
    opts = []
    for c in range(args.clouds):
        _, params = R.pack(S.make_params_device(cfg, dev))
        _, grads = R.pack(S.grads_device(cfg, 0, dev))
        o = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5,
                    errors="ignore", fused_compaction=args.fused)
        opts.append((o, grads))
    vis = S.visibility_device(cfg, 0, dev)
    trace = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
    for rep in range(3):
        for j, (o, g) in enumerate(opts):
            last = rep == 2 and j == len(opts) - 1
            if last:
                torch.cuda.synchronize()
                lib.gs_debug_set_trace(trace.data_ptr())
            o.step(vis, 1_000_000, grads=g)
            if last:
                torch.cuda.synchronize()
                lib.gs_debug_set_trace(None)
    t = trace.view(4096, 16).cpu().numpy().astype(np.int64)
    live = t[:, 0] > 0
    t = t[live]
    t0 = t[:, 0].min()
    two_phase = (t[:, 13] > 0).any()  # slot 13: the grid-barrier stamp
    print(f"rows {args.rows} vis {args.vis} fused {args.fused} two-phase {two_phase}: {live.sum()} CTAs, "
          f"visible {t[:, 9].sum()}, kernel span {(t[:, 11].max() - t0) / 1e3:.2f} us")
    rel = lambda k: (t[:, k] - t0) / 1e3  # noqa: E731
    names = dict(NAMES)
    if two_phase:
        names = {0: "entry", 12: "phase A done", 13: "grid barrier",
                 **{k: v for k, v in NAMES.items() if k}}
    for k, name in names.items():
        x = rel(k)
        print(f"  {k:2d} {name:16s} min {x.min():7.2f}  p50 {np.median(x):7.2f}  "
              f"p90 {np.percentile(x, 90):7.2f}  max {x.max():7.2f} us")
    lastb = t[:, 7] > 0
    if lastb.any():
        print(f"   7 final reduce in  {rel(7)[lastb][0]:7.2f}   8 final reduce out {rel(8)[lastb][0]:7.2f}")
    if not two_phase:  # slots 12, 14, 15: loader cycles, waits on a free stage / mask tiles
        cyc = t[:, 12].astype(np.float64)
        ok = cyc > 0
        if ok.any():
            print(f"  loader cycles p50 {np.median(cyc[ok]):.0f}; waiting on a free stage "
                  f"{np.median(t[ok, 14] / cyc[ok]) * 100:.1f}% / on mask tiles "
                  f"{np.median(t[ok, 15] / cyc[ok]) * 100:.1f}% (p50 over CTAs)")
    work = t[:, 9]
    dur = (t[:, 4] - t[:, 3]) / 1e3
    print(f"  rows per CTA: min {work.min()} max {work.max()} mean {work.mean():.1f}; "
          f"consumer busy p50 {np.median(dur):.2f} max {dur.max():.2f} us")
    order = np.argsort(t[:, 11])[-5:]
    print("  last CTAs to exit: rows", work[order].tolist(), "exit",
          np.round(rel(11)[order], 2).tolist(), "entry", np.round(rel(0)[order], 2).tolist())


if __name__ == "__main__":
    main()
