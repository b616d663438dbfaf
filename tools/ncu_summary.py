"""Summarise an ncu report (raw metrics + hottest stall sites) -- reading aid."""
import csv
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def main(rep, top=8):
    hdr, units, rows = raw(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct",
            "smsp__issue_active.avg.pct", "sm__warps_active.avg.pct", "launch__grid_size",
            "launch__cluster_dim_x", "launch__block_size", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "lts__t_sectors_srcunit_tex_op_read.sum", "launch__shared_mem_per_block_dynamic"]
    for row in rows:
        print("=====", row[hdr.index("Kernel Name")][:70])
        for i, h in enumerate(hdr):
            if any(h.startswith(k) for k in keys) and not h.endswith("per_second"):
                print(f"  {h} = {row[i]} {units[i]}")
        st = [(h, row[i]) for i, h in enumerate(hdr)
              if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and row[i]]
        st = sorted(st, key=lambda x: -float(x[1].replace(",", "")))[:8]
        print("  stalls:", ", ".join(f"{h.split('stalled_')[1]}={v}" for h, v in st))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    lines = out.splitlines()
    blocks, cur = [], None
    for l in lines:
        if l.startswith('"Kernel Name"'):
            cur = [l]
            blocks.append(cur)
        elif cur is not None and l.strip():
            cur.append(l)
    for b in blocks:
        rr = list(csv.reader(b[1:]))
        h = rr[0]
        si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        data = [(r[1].strip(), int(r[si] or 0), int(r[ei] or 0)) for r in rr[1:] if len(r) > si]
        tot = max(sum(d[1] for d in data), 1)
        print("  total warp-instr executed", sum(d[2] for d in data))
        for i in sorted(range(len(data)), key=lambda i: -data[i][1])[:top]:
            ctx = " | ".join(d[0][:38] for d in data[max(0, i - 3):i])
            print(f"  {100 * data[i][1] / tot:5.1f}%  {data[i][0][:40]:40s}  <- {ctx}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8)
