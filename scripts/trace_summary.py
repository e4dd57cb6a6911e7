"""Summarise an AO Chrome trace (ao_ctx_trace_dump): per role busy time, chunk-wait time,
transfer completion times, reduction tail -- one block per kernel launch.
usage: python scripts/trace_summary.py TRACE.json [LAUNCH]"""
import collections
import json
import sys


def summarise(ev):
    t0 = min(e["ts"] for e in ev)
    for e in ev:
        e["ts"] -= t0
    t_end = max(e["ts"] + e["dur"] for e in ev)
    print(f"events {len(ev)}, span {t_end:.1f} us")
    by = collections.defaultdict(list)
    for e in ev:
        by[e["cat"]].append(e)
    for k, es in sorted(by.items()):
        durs = [e["dur"] for e in es]
        ends = sorted(e["ts"] + e["dur"] for e in es)
        starts = sorted(e["ts"] for e in es)
        # time-sliced launches: one physical CTA serves every rank (same tid under several pids)
        ts = len({e["pid"] for e in ev}) > 1 and any(
            len({x["pid"] for x in ev if x["tid"] == t}) > 1 for t in {e["tid"] for e in ev[:200]})
        lanes = len({e["tid"] for e in es}) if ts else len({(e["pid"], e["tid"]) for e in es})
        print(f"  {k:12s} n={len(es):6d} lanes={lanes:4d} mean={sum(durs) / len(durs):8.2f}us max={max(durs):8.2f}us "
              f"first={starts[0]:8.1f} last_end={ends[-1]:8.1f} busy/lane={sum(durs) / max(lanes, 1) / t_end:6.1%}")
    if by.get("wait"):
        w = sorted(by["wait"], key=lambda e: -e["dur"])[:4]
        print("  longest waits:", [(e["pid"], e["tid"] // 8, e["name"], round(e["dur"], 1), round(e["ts"], 1)) for e in w])
    if by.get("mma"):
        first = min(e["ts"] for e in by["mma"])
        print(f"  first mma start {first:.1f}, last mma end {max(e['ts'] + e['dur'] for e in by['mma']):.1f}")


def main():
    ev_all = json.load(open(sys.argv[1]))["traceEvents"]
    if not ev_all:
        sys.exit("no events")
    sel = int(sys.argv[2]) if len(sys.argv) > 2 else None
    launches = sorted({e.get("args", {}).get("launch", 0) for e in ev_all})
    tmin = min(e["ts"] for e in ev_all)
    for L in launches:
        if sel is not None and L != sel:
            continue
        ev = [dict(e) for e in ev_all if e.get("args", {}).get("launch", 0) == L]
        start = min(e["ts"] for e in ev) - tmin
        print(f"=== launch {L} (starts at {start:.1f} us)")
        summarise(ev)


if __name__ == "__main__":
    main()
