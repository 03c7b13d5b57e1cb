"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def summarize(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        tot[k] += float(d["Metric Value"])
        cnt[k] += 1
    T = sum(tot.values())
    lines = [f"{'kernel':42s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>9s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        lines.append(f"{k:42s} {cnt[k]:8d} {v / 1e6:9.2f} {v / T * 100:5.1f}% {v / cnt[k] / 1e3:9.1f}")
    lines.append(f"{'TOTAL':42s} {sum(cnt.values()):8d} {T / 1e6:9.2f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
