"""Remote-traffic timeline of one traced cycle of the xfer kernel (GR_TRACE output): per 5-us bin,
the NVLink bytes/s implied by the active reduce-scatter and all-gather items (each item's
remote bytes spread uniformly over its ready->done span) and the number of active items.

  python tools/trace_timeline.py gpurun_out/tr64.rank0.jsonl [--cycle 1] [--N 4] [--bin 5]
"""
import argparse
import collections
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--cycle", type=int, default=1)
    ap.add_argument("--N", type=int, default=4)
    ap.add_argument("--pb", type=int, default=2)
    ap.add_argument("--bin", type=float, default=5.0)
    a = ap.parse_args()
    recs = [json.loads(l) for l in open(a.path)]
    r = recs[a.cycle]
    items = r["items"]
    C = r["nitems"] // 3
    ce = r["elems"] / C
    remote = {0: 0.0, 1: (a.N - 1) * ce * a.pb, 2: ce * a.pb}
    t0 = min(x[1] for x in items)
    bins = collections.defaultdict(float)
    active = collections.defaultdict(collections.Counter)
    end = 0.0
    for it, g, rd, dn, cs in items:
        ph = min(2, it // C)
        s, e = (rd - t0) / 1e3, (dn - t0) / 1e3
        end = max(end, e)
        if e <= s:
            continue
        rate = remote[ph] / (e - s)
        b = int(s // a.bin)
        while b * a.bin < e:
            lo, hi = max(s, b * a.bin), min(e, (b + 1) * a.bin)
            bins[b] += rate * (hi - lo)
            active[b][ph] += 1
            b += 1
    tot = sum(remote[min(2, x[0] // C)] for x in items)
    print(f"cycle {a.cycle}: span {end:.1f} us, remote {tot / 1e6:.1f} MB -> {tot / end / 1e3:.1f} GB/s average")
    for b in sorted(bins):
        print(f"{b * a.bin:6.0f}-{(b + 1) * a.bin:6.0f} us: remote {bins[b] / a.bin / 1e3:6.1f} GB/s  "
              f"active pack/rs/ag {active[b][0]:3d} {active[b][1]:3d} {active[b][2]:3d}")


if __name__ == "__main__":
    main()
