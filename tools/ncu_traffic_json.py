"""Per-launch DRAM traffic of the mm2 / adjoint GEMM from an ncu capture of
tools/gemm_shapes.py (tools/ncu_traffic.sh): writes the JSON bench.py
quotes as roofline.traffic.  python tools/ncu_traffic_json.py REP OUT"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, units, rows = raw[0], raw[1], raw[2:]


def col(name):
    return h.index(name)


d, f, T = 2048, 5632, 8192
order = [("mm2", d, d, 4), ("adjoint", d, d, 4), ("mm2", d, f, 2), ("adjoint", d, f, 2), ("mm2", f, d, 1),
         ("adjoint", f, d, 1)]
shapes = []
for r, (op, m, n, per) in zip(rows, order):
    def val(name):
        v = float(r[col(name)].replace(",", ""))
        u = units[col(name)]
        return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)
    us = float(r[col("gpu__time_duration.sum")].replace(",", "")) * (1e-3 if units[col("gpu__time_duration.sum")] == "nsecond" else 1.0)
    shapes.append({"op": op, "m": m, "n": n, "T": T, "launches_per_layer": per, "time_us": us,
                   "dram_read_bytes": val("dram__bytes_read.sum"), "dram_write_bytes": val("dram__bytes_write.sum"),
                   "l2_to_sm_bytes": val("l1tex__m_xbar2l1tex_read_bytes.sum"),
                   "tensor_pipe_active_pct": float(r[col("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")]),
                   "tflops": 2.0 * T * m * n / (us * 1e-6) / 1e12})
w = sum(s["launches_per_layer"] for s in shapes)
traffic = sum((s["dram_read_bytes"] + s["dram_write_bytes"]) * s["launches_per_layer"] for s in shapes) / w
json.dump({"kernel": "tc2_kernel (CTA-pair tcgen05 GEMM: mm2 and adjoint; 512x256 pair tiles at T = 8192)",
           "command": "ncu --set full --clock-control none -k regex:tc2_kernel python tools/gemm_shapes.py "
                      "(B200, one launch per Llama-1B projection shape and direction, T=8192)",
           "traffic_bytes_per_launch": traffic,
           "note": "launch-weighted over the 7 projections of a decoder block; DRAM writes of the output partly "
                   "stay in L2 at kernel end",
           "shapes": shapes}, open(out, "w"), indent=1)
print(out, traffic)
