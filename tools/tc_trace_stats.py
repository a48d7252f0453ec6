"""Per-role summary of a BX_TC_TRACE timeline (tools/tc_trace.py / tools/large_n.py LARGE_N_TRACE):
MMA waits for the producers and per-pass issue spans, epilogue drain / wait per chunk, producer slot
waits.  python tools/tc_trace_stats.py FILE..."""
import sys

import numpy as np


def stats(f):
    t = np.fromfile(f, dtype=np.int64).reshape(4, 4096, 2)
    t0 = min(int(t[r, 0, 0]) for r in range(4) if t[r, 0, 0])
    ev = {r: t[r][t[r, :, 0] != 0] for r in range(4)}
    m = ev[1]
    codes, clk = m[:, 1] >> 16, m[:, 0] - t0
    waits, spans, last_ok, w = [], [], None, 0
    for i in range(len(m)):
        if codes[i] == 1:
            if last_ok is not None:
                spans.append(clk[i] - last_ok)
            w = clk[i]
        elif codes[i] == 2:
            waits.append(clk[i] - w)
            last_ok = clk[i]
    e = ev[2]
    ec, eclk = e[:, 1] >> 16, e[:, 0] - t0
    dr = [eclk[i] - eclk[i - 1] for i in range(1, len(e)) if ec[i] == 2 and ec[i - 1] == 1]
    wt = [eclk[i] - eclk[i - 1] for i in range(1, len(e)) if ec[i] == 1 and ec[i - 1] == 2]
    p = ev[0]
    pc, pclk = p[:, 1] >> 16, p[:, 0] - t0
    sw = [pclk[i] - pclk[i - 1] for i in range(1, len(p)) if pc[i] == 4 and pc[i - 1] == 3]
    starts = clk[codes == 2]
    print(f"{f}: mma passes {len(waits)}, wait-for-producers mean {np.mean(waits[1:]):.0f} clk, "
          f"issue span mean {np.mean(spans):.0f}; epilogue drain mean {np.mean(dr):.0f} / wait mean "
          f"{np.mean(wt):.0f} clk over {len(dr)} chunks; producer slot wait mean {np.mean(sw):.0f}")


if __name__ == "__main__":
    for f in sys.argv[1:]:
        stats(f)
