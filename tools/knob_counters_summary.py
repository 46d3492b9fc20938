"""Join tools/knob_counters.py's plain JSON lines with the ncu CSV of the same run order
(BATCHES captured k_gather_mean_row launches per knob point) -> one JSON summary."""
import csv
import io
import json
import sys


def main(plain_path, ncu_csv, peak_gbs=6538.9):
    pts = [json.loads(l) for l in open(plain_path) if l.startswith("{")]
    rows = list(csv.reader(io.StringIO("".join(l for l in open(ncu_csv) if not l.startswith("==")))))
    h = rows[0]
    data = [dict(zip(h, r)) for r in rows[1:]]
    # long format: one row per (launch, metric)
    by_id = {}
    for d in data:
        if "Metric Name" not in d:
            continue
        by_id.setdefault(int(d["ID"]), {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    launches = [by_id[k] for k in sorted(by_id)]
    out = []
    i = 0
    for p in pts:
        n, w = p["batches"], p.get("warm", 0)
        ls = launches[i + w: i + w + n]
        i += w + n
        def mean(key, scale=1.0):
            v = [float(x[key][0].replace(",", "")) * scale for x in ls if key in x]
            return sum(v) / len(v) if v else None
        unit = ls[0]["gpu__time_duration.sum"][1] if ls else "ns"
        t_scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1e-9)
        bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        t = mean("gpu__time_duration.sum", t_scale)
        rd = mean("dram__bytes_read.sum", bscale.get(ls[0]["dram__bytes_read.sum"][1], 1))
        wr = mean("dram__bytes_write.sum", bscale.get(ls[0]["dram__bytes_write.sum"][1], 1))
        q = dict(p)
        q.update({"ncu_gather_us": t * 1e6, "ncu_dram_read_bytes": rd, "ncu_dram_write_bytes": wr,
                  "ncu_dram_gbps": (rd + wr) / t / 1e9,
                  "ncu_dram_frac_of_peak": (rd + wr) / t / 1e9 / peak_gbs,
                  "algorithmic_gbps_under_ncu": p["algorithmic_bytes"] / t / 1e9,
                  "l2_hit_rate_pct": mean("lts__t_sector_hit_rate.pct"),
                  "dram_read_over_unique_bytes": rd / p["unique_feature_bytes"]})
        out.append(q)
    print(json.dumps({"peak_gbs": peak_gbs, "points": out}, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:3])
