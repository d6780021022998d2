"""Per-iteration DRAM traffic of the CRVPINN iteration per workload, from ncu --set full captures of one
eager loss_grad (scripts/prof_once.py <cfg> 1; every kernel of A1-A7 once): the sum over those kernels of
dram__bytes_read.sum + dram__bytes_write.sum -> profiles/r02_traffic.json (read by bench.py).
usage: python scripts/ncu_traffic.py C5=gpurun_out/r02_full_c5.ncu-rep C4=... [out.json]"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def kernel_bytes(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    out = []
    for d in data:
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[ix[m]]) * SCALE.get(units[ix[m]], 1.0)
        out.append((d[ix["Kernel Name"]].split("(")[0].replace("void ", ""), b))
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if "=" in a]
    outp = next((a for a in sys.argv[1:] if a.endswith(".json")), "profiles/r02_traffic.json")
    res = {"bytes_per_iter": {}, "kernels": {},
           "source": "ncu --set full --clock-control none, one eager loss_grad per workload (scripts/prof_once.py); "
                     "sum of dram__bytes_read.sum + dram__bytes_write.sum over its kernels (A1-A7; the Adam "
                     "update rides on the reductions in the timed graph and is not in this sum); cold L2"}
    for a in args:
        name, rep = a.split("=", 1)
        kb = kernel_bytes(rep)
        res["bytes_per_iter"][name] = sum(b for _, b in kb)
        res["kernels"][name] = [[k, b] for k, b in kb]
    with open(outp, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res["bytes_per_iter"]))
