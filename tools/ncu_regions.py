"""Summarize an ncu report: headline metrics + stall samples per barrier-delimited region."""
import csv, subprocess, sys
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
for line in det.splitlines():
    if any(k in line for k in ["Duration", "DRAM Throughput", "L2 Hit Rate", "Eligible Warps", "No Eligible", "Achieved Occupancy", "Registers Per", "Issue Slots Busy", "Dynamic Shared"]):
        print(line.strip())
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
if len(rows) > 2:
    h, v = rows[0], rows[2]
    for name in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum"]:
        if name in h:
            print(name, v[h.index(name)], rows[1][h.index(name)])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; idx = {x: i for i, x in enumerate(hdr)}; data = rows[2:]
key = "Warp Stall Sampling (All Samples)"; ex = "Instructions Executed"
stall_cols = [x for x in hdr if x.startswith('stall_') and 'Not Issued' not in x]
tot = sum(int(r[idx[key]] or 0) for r in data)
agg = {c: sum(int(r[idx[c]] or 0) for r in data) for c in stall_cols}
print("samples", tot, sorted(((v, k) for k, v in agg.items()), reverse=True)[:8])
acc = 0; start = data[0][idx['Address']][-5:]
for i, r in enumerate(data):
    s = r[idx['Source']]
    acc += int(r[idx[key]] or 0)
    if 'BAR.SYNC' in s or 'TRYWAIT' in s or i == len(data) - 1:
        print(f"  {start}..{r[idx['Address']][-5:]} {acc:7d} ({100*acc/max(tot,1):4.1f}%) -> {s.strip()[:40]} x{r[idx[ex]]}")
        acc = 0; start = data[i + 1][idx['Address']][-5:] if i + 1 < len(data) else ''
top = sorted(data, key=lambda r: -int(r[idx[key]] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for r in top:
    st = sorted(((int(r[idx[c]] or 0), c) for c in stall_cols), reverse=True)[:2]
    print(f"{int(r[idx[key]] or 0):6d} {r[idx['Address']][-5:]} {r[idx['Source']][:64]:64s} {st}")
