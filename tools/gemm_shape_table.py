"""Per-shape GEMM roofline table from an `ncu --set full` capture of
tools/gemm_shapes.py (exported with `ncu -i REP --page raw --csv`): duration,
achieved TFLOP/s, tensor-pipe activity, DRAM bytes against the algorithmic
bytes of the shape (A and B read once, C written once in its dtype, plus the
epilogue's row operand / fp32 accumulator).

    python tools/gemm_shape_table.py RAW.csv SHAPES.log OUT.json
"""
import ast
import csv
import json
import sys


TP = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    raw, shapes_log, out = sys.argv[1:4]
    shapes = []
    for line in open(shapes_log):
        if "(" in line:
            name, tup = line.split(" (", 1)
            shapes.append((name.strip(), ast.literal_eval("(" + tup.strip())))
    rows = list(csv.reader(open(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, k):
        v = num(r[col[k]])
        u = units[col[k]].lower()
        scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-3,
                 "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
        return None if v is None else v * scale

    table = []
    launches = [r for r in data if "gemm_tc" in r[col["Kernel Name"]]]
    for (name, (M, N, K, amn, bmn, epi)), r in zip(shapes, launches):
        dur = get(r, "gpu__time_duration.sum")   # us
        rd, wr = get(r, "dram__bytes_read.sum"), get(r, "dram__bytes_write.sum")
        a_b = 2 * (M * K + N * K)
        c_b = {0: 2, 1: 2, 2: 2, 3: 4, 4: 2, 5: 8, 6: 4}[epi] * M * N
        extra = {2: 2 * M * N, 4: 2 * M * N}.get(epi, 0)
        alg = a_b + c_b + extra
        table.append({"gemm": name, "M": M, "N": N, "K": K, "epilogue": epi,
                      "duration_us": round(dur, 2),
                      "tflops": round(2.0 * M * N * K / (dur * 1e-6) / 1e12, 1),
                      "tensor_pipe_pct": get(r, TP) if TP in col else None,
                      "dram_mb": round((rd + wr) / 1e6, 1), "algorithmic_mb": round(alg / 1e6, 1),
                      "dram_over_algorithmic": round((rd + wr) / alg, 3)})
    json.dump({"source": "ncu --set full of tools/gemm_shapes.py (one launch per shape, warm "
                         "round skipped), --clock-control none", "shapes": table},
              open(out, "w"), indent=1)
    for t in table:
        print(t)


if __name__ == "__main__":
    main()
