"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel:
launch count, mean / min device time and share of the profiled total.
Launch times under ncu are cold-cache and serialised: compare shares."""
import collections
import csv
import sys


def main(path: str, skip_prefix: tuple = ("k_transpose_shard", "fb::k_init", "fb::k_peak", "<unnamed>::k_b_")) -> None:
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = d["Kernel Name"].split("(")[0].replace("void ", "")
            agg.setdefault(k, []).append(float(d["Metric Value"]) / 1e3)
    round_k = {k: v for k, v in agg.items() if not k.startswith(skip_prefix)}
    tot = sum(sum(v) for v in round_k.values())
    print(f"{'kernel':34s} {'launches':>8s} {'mean us':>9s} {'min us':>9s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = sum(v) / tot if k in round_k else float("nan")
        print(f"{k:34s} {len(v):8d} {sum(v)/len(v):9.1f} {min(v):9.1f} {share:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
