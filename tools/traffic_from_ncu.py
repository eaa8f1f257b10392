"""Write profiles/traffic.json: DRAM bytes per launch (dram__bytes_read.sum + write) of each
kernel in an `ncu --set full` report, for bench.py's roofline `traffic` field.
usage: python tools/traffic_from_ncu.py REPORT.ncu-rep [REPORT2 ...]"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME_MS = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main():
    out = {}
    for rep in sys.argv[1:]:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        hdr, units = rows[0], rows[1]
        ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        it, ik = hdr.index("gpu__time_duration.sum"), hdr.index("Kernel Name")
        for r in rows[2:]:
            name = r[ik].split("(")[0].split("::")[-1].split("<")[0].strip()
            b = float(r[ir]) * UNIT[units[ir]] + float(r[iw]) * UNIT[units[iw]]
            out[name] = {"dram_bytes_per_launch": b, "ncu_ms": float(r[it]) * TIME_MS.get(units[it], 1.0),
                         "report": os.path.basename(rep)}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    path = os.path.join(root, "profiles", "traffic.json")
    # stamped with the kernel sources' hash: bench.py refuses a capture of other kernels
    json.dump({"sources_sha": bench.sources_sha(), "kernels": out}, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
