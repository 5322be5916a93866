"""Summarise an `ncu --set full` capture of gemm_tc launches (exported with
`ncu -i REP --page raw --csv`) into profiles/ncu_gemm_summary.json: per-launch
duration, DRAM bytes, tensor-pipe and throughput percentages, and the mean
DRAM bytes per launch that bench.py reports as roofline.traffic.

    python tools/ncu_gemm_summary.py RAW.csv OUT.json "source description"
"""
import csv
import json
import sys


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    raw, out, source = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(open(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, k, scale_to_bytes=False):
        if k not in col:
            return None
        v = num(r[col[k]])
        if v is None or not scale_to_bytes:
            return v
        u = units[col[k]].lower()
        return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)

    launches = []
    for r in data:
        if "gemm_tc" not in r[col["Kernel Name"]]:
            continue
        dur = get(r, "gpu__time_duration.sum")
        if units[col["gpu__time_duration.sum"]].lower().startswith("n"):
            dur = dur / 1e3
        elif units[col["gpu__time_duration.sum"]].lower().startswith("m"):
            dur = dur * 1e3
        launches.append({
            "kernel": r[col["Kernel Name"]].split("(")[0],
            "grid": r[col["launch__grid_size"]] if "launch__grid_size" in col else None,
            "duration_us": dur,
            "dram_read_bytes": get(r, "dram__bytes_read.sum", True),
            "dram_write_bytes": get(r, "dram__bytes_write.sum", True),
            "tensor_pipe_pct": get(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            "sm_throughput_pct": get(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram_throughput_pct": get(r, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "registers": r[col["launch__registers_per_thread"]] if "launch__registers_per_thread" in col else None,
        })
    tot = [l["dram_read_bytes"] + l["dram_write_bytes"] for l in launches
           if l["dram_read_bytes"] is not None and l["dram_write_bytes"] is not None]
    summary = {"source": source, "launches": launches,
               "dram_bytes_per_launch": sum(tot) / len(tot) if tot else None}
    json.dump(summary, open(out, "w"), indent=1)
    print(f"{len(launches)} launches, mean DRAM bytes/launch {summary['dram_bytes_per_launch']}")


if __name__ == "__main__":
    main()
