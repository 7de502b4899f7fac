"""Summarise GR_TRACE output (<prefix>.rank<r>.jsonl): bitvector-kernel phases,
host hand-off, and per-phase item timings of the fused data kernel.

  python tools/trace_summary.py gpurun_out/trace [--chrome out.json]
"""
import argparse
import glob
import json
import statistics as st


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(q * len(xs)))] if xs else float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("prefix")
    ap.add_argument("--chrome")
    a = ap.parse_args()
    events = []
    for path in sorted(glob.glob(a.prefix + ".rank*.jsonl")):
        recs = [json.loads(l) for l in open(path)]
        print(f"== {path}: {len(recs)} cycles")
        kpop = [(r["k"][1] - r["k"][0]) / 1e3 for r in recs]
        kand = [(r["k"][2] - r["k"][1]) / 1e3 for r in recs]
        krel = [(r["k"][3] - r["k"][2]) / 1e3 for r in recs]
        h = [r["h"] for r in recs]  # [enter, snapshot taken, bitvector launched, all launched, seen, done]
        hs = [(x[1] - x[0]) / 1e3 for x in h]
        hb = [(x[2] - x[1]) / 1e3 for x in h]
        hl = [(x[3] - x[2]) / 1e3 for x in h]
        hw = [(x[4] - x[3]) / 1e3 for x in h]
        hd = [(x[5] - x[4]) / 1e3 for x in h]
        print(f"  bitvector kernel us: populate p50 {pct(kpop,.5):.2f}  AND p50 {pct(kand,.5):.2f}  "
              f"release+handoff p50 {pct(krel,.5):.2f}")
        print(f"  host us p50: entry+snapshot {pct(hs,.5):.2f}  bitvector launch {pct(hb,.5):.2f}  "
              f"data launch {pct(hl,.5):.2f}  wait-for-handoff {pct(hw,.5):.2f}  decode {pct(hd,.5):.2f}")
        for r in recs:
            raw = r["items"]
            if not raw:
                continue
            # [item, grab, ready, done, cta|smid] (items never executed are omitted)
            n = max(r.get("nitems", 0), max(x[0] for x in raw) + 1)
            it = [[0, 0, 0, 0] for _ in range(n)]
            for x in raw:
                it[x[0]] = x[1:]
            if r.get("prof"):
                pf = [x for x in r["prof"] if x[0]]
                if pf:
                    tot = sum(x[0] for x in pf)
                    ctot = sum(x[3] for x in pf) or 1
                    print(f"    producer: ring-full stalls {100 * sum(x[1] for x in pf) / tot:.1f}%, "
                          f"flag waits {100 * sum(x[2] for x in pf) / tot:.1f}% | consumers: starved (ring empty) "
                          f"{100 * sum(x[4] for x in pf) / ctot:.1f}%, flag publish {100 * sum(x[5] for x in pf) / ctot:.1f}%")
            live = [x for x in it if x[0]]
            if not live:
                continue
            t0 = min(x[0] for x in live)
            t1 = max(x[2] for x in live)
            ctas = len({x[3] & 0xffffffff for x in live})
            print(f"  cycle {r['cycle']} algo {r['algo']} elems {r['elems']} items {len(it)} ctas {ctas} "
                  f"span {(t1 - t0) / 1e3:.1f} us  (kernel-start -> first grab {(t0 - r['k'][3]) / 1e3:.1f} us after bv end)")
            nph = {1: 1, 2: 2, 3: 3, 4: 3}.get(r["algo"], 1)
            per = max(1, len(it) // nph)
            for ph in range(nph):
                seg = [x for x in it[ph * per:(ph + 1) * per] if x[0] and x[2]]
                if not seg:
                    continue
                dur = [(x[2] - x[0]) / 1e3 for x in seg]
                wait = [(x[1] - x[0]) / 1e3 for x in seg if x[1]]
                work = [(x[2] - x[1]) / 1e3 for x in seg if x[1]]
                s0 = (min(x[0] for x in seg) - t0) / 1e3
                s1 = (max(x[2] for x in seg) - t0) / 1e3
                line = f"    phase {ph}: {len(seg)} items, window {s0:.1f}..{s1:.1f} us, item p50 {pct(dur,.5):.2f} p90 {pct(dur,.9):.2f} us"
                if wait:
                    line += f", wait p50 {pct(wait,.5):.2f} p90 {pct(wait,.9):.2f}, work p50 {pct(work,.5):.2f}"
                print(line)
                if a.chrome:
                    for x in seg:
                        events.append({"name": f"ph{ph}", "ph": "X", "ts": x[0] / 1e3, "dur": (x[2] - x[0]) / 1e3,
                                       "pid": r["rank"], "tid": x[3] & 0xffffffff})
            if a.chrome:
                events.append({"name": "bitvector", "ph": "X", "ts": r["k"][0] / 1e3,
                               "dur": (r["k"][3] - r["k"][0]) / 1e3, "pid": r["rank"], "tid": -1})
    if a.chrome:
        json.dump({"traceEvents": events}, open(a.chrome, "w"))


if __name__ == "__main__":
    main()
