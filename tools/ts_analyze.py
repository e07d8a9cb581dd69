"""Summarise per-tile timestamps of CTA 0 (SPCP_TC_TIMESTAMPS build, SPCP_TC_DEBUG=4).
Columns: 0 X issued, 1 residual issued, 2 MMA saw ga_full, 3 MMA passed gt_empty,
4 epi top, 5 s_full seen, 6 stage_full seen, 7 math done, 8 drains done,
9 ga/gs waits done, 10 ga_full arrive, 11 V copy start, 12 residual u_full ok, 13 v_full ok."""
import sys
import numpy as np

rows = [list(map(int, l.split())) for l in open(sys.argv[1]) if l.strip()]
a = np.array(rows, dtype=float)
a[a < 0] = np.nan
s = slice(8, 60)
def d(i, j, lag=0, name=""):
    x = a[s, j] - (a[s.start - lag:s.stop - lag, i] if lag else a[s, i])
    print(f"{name:44s} median {np.nanmedian(x):8.0f}  mean {np.nanmean(x):8.0f}")
print("period per tile (epi top t -> t+2)/2     ", np.nanmedian((a[10:60, 4] - a[8:58, 4]) / 2))
d(4, 5, name="epi: wait S (top -> s_full)")
d(5, 6, name="epi: wait X after S")
d(6, 7, name="epi: math")
d(7, 8, name="epi: drains (incl. gt_full wait)")
d(8, 9, name="epi: ga/gs waits + tmem st")
d(9, 10, name="epi: STS + fence + arrive")
d(1, 5, name="residual issue -> s_full seen")
d(10, 2, name="ga_full arrive (warp3/7) -> MMA sees it")
d(2, 3, name="MMA: ga_full -> gt_empty ok")
d(11, 13, name="V copy start -> MMA v_full ok")
d(13, 1, name="MMA: v_full -> s_empty ok (residual issue)")
d(0, 6, name="X issue -> epi sees stage_full")
if a.shape[1] >= 24:
    print("per-warp ga_full arrival relative to warp (q=0,h=0) [quarter q on SMSP (q+3)%4]:")
    base = a[s, 16]
    for h in range(2):
        print("  h=%d: " % h + "  ".join("q%d %6.0f" % (q, np.nanmedian(a[s, 16 + q + 4 * h] - base)) for q in range(4)))
    d(23, 14, name="last warp arrival -> MMA reductions start")
    last = np.nanmax(a[s, 16:24], axis=1)
    x = a[s, 2] - last
    print("last arrival -> MMA saw ga_full           median", np.nanmedian(x))
    x = a[s, 14] - last
    print("last arrival -> MMA entered reductions()  median", np.nanmedian(x))
if a.shape[1] >= 26:
    d(1, 24, name="MMA: residual issue (6 MMAs + commit)")
    d(3, 25, name="MMA: GtU issue (16 MMAs + 2 commits)")
    d(25, 15, name="MMA: GV issue (8 MMAs + commits)")
