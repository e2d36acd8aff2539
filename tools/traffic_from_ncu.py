"""Regenerate profiles/traffic.json from the full-batch ncu --set full
captures of a measurement pass (tools/gpu_full_measure.sh): DRAM bytes per
launch (dram__bytes_read.sum + dram__bytes_write.sum) per image, next to the
kernel's compulsory bytes (the algorithmic bytes bench.py's roofline uses).

    python tools/traffic_from_ncu.py gpurun_out/r2final [out.json]
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2002_00552_b200 import _native  # noqa: E402
from paper_2002_00552_b200.configs import WORKLOADS  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
KERNEL = {"tc": "gemm_output", "it": "input_transform", "sc": "conv2d_small_c"}


def metrics(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            d[h] = float(v.replace(",", "")) * UNIT.get(u, 1)
        except ValueError:
            pass
    return d


def compulsory(kind, wl):
    spec = wl.spec()
    desc = _native.make_desc(wl.batch, wl.c_in, wl.hw, wl.hw, wl.c_out, spec.kernel, spec.stride, spec.pad)
    x = 4.0 * wl.batch * wl.c_in * wl.hw * wl.hw
    y = 4.0 * wl.batch * wl.c_out * desc.oh * desc.ow
    v = 4.0 * desc.num_freqs * desc.tiles * wl.c_in
    u = 4.0 * desc.num_freqs * wl.c_out * wl.c_in
    # tc: U is the stacked fp16 hi/lo split (2 x 2 bytes per fp32 value)
    return {"tc": v + u + y, "it": x + v, "sc": x + u + y}[kind]


def main():
    src = Path(sys.argv[1])
    out = {}
    for rep in sorted(src.glob("ncu_*_cfg*.ncu-rep")):
        kind, name = rep.stem.split("_", 2)[1:]
        wl = WORKLOADS[name]
        m = metrics(rep)
        traffic = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        comp = compulsory(kind, wl)
        out.setdefault(name, {})[KERNEL[kind]] = {
            "bytes_per_image": traffic / wl.batch, "batch": wl.batch,
            "dram_read": m["dram__bytes_read.sum"], "dram_write": m["dram__bytes_write.sum"],
            "compulsory_bytes": comp, "traffic_over_compulsory": traffic / comp,
            "kernel_ms_under_ncu": m.get("gpu__time_duration.sum", 0) * 1e3 if m.get("gpu__time_duration.sum", 1) < 1 else None,
            "capture": f"profiles/r2/{rep.stem}.txt (full batch, ncu --set full)",
            "note": ("writes below the compulsory bytes = dirty lines still in the 126 MB L2 at kernel end"
                     if m["dram__bytes_write.sum"] < comp and kind != "tc" else ""),
        }
    dst = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "profiles" / "traffic.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    for name, ks in out.items():
        for k, e in ks.items():
            print(f"{name:22s} {k:16s} traffic/compulsory {e['traffic_over_compulsory']:.3f}")


if __name__ == "__main__":
    main()
