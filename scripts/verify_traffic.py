"""Summarise ncu launch lists of one eager verify forward (scripts/ncu_verify.py b k) into
profiles/verify_traffic.json: DRAM bytes read + written over the forward's kernels, per (b, k).
python scripts/verify_traffic.py out.json b:k:csv [b:k:csv ...]"""
import csv, json, sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    per = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1,
             "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        d = per.setdefault(r[ix["ID"]], {})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1)
    tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in per.values())
    us = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())
    return len(per), tot, us


out = sys.argv[1]
entries = []
for spec in sys.argv[2:]:
    b, k, path = spec.split(":", 2)
    n, tot, us = summarise(path)
    entries.append({"workload": "llama-2-7b verify forward", "b": int(b), "k": int(k), "ctx": 192,
                    "dram_bytes_read_plus_write": int(tot), "kernels": n, "serialised_us": round(us, 1),
                    "source": "ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                              "dram__bytes_write.sum --clock-control none python scripts/ncu_verify.py "
                              f"{b} {k} (one eager forward, engine-autotuned GEMM plans); {path.split('/')[-1]}"})
json.dump({"entries": entries}, open(out, "w"), indent=1)
print(json.dumps(entries, indent=1))
