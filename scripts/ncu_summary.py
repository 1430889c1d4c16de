"""Summarise ncu --set full reports (one kernel each): duration, DRAM bytes, tensor-pipe activity, registers,
occupancy and the top warp-stall reasons; optionally the hottest source lines.
usage: python scripts/ncu_summary.py REPORT.ncu-rep [...] [--lines N]"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration (us)"), ("dram__bytes_read.sum", "dram read (MB)"),
        ("dram__bytes_write.sum", "dram write (MB)"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
        ("launch__registers_per_thread", "registers"), ("launch__grid_size", "grid"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %")]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    units = dict(zip(h, rows[1]))
    return [(dict(zip(h, r)), units) for r in rows[2:]]


def conv(k, v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    scale = {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}
    if "time" in k:
        return round(x * scale.get(unit, 1), 3)
    if "bytes" in k:
        return round(x * scale.get(unit, 1e-6), 3)
    return round(x, 2)


def main():
    args = sys.argv[1:]
    nlines = 0
    if "--lines" in args:
        i = args.index("--lines")
        nlines = int(args[i + 1])
        del args[i:i + 2]
    for rep in args:
        for d, units in raw(rep):
            name = d.get("Kernel Name", "?")[:90]
            print(f"## {rep.split('/')[-1]}: {name}")
            for k, label in KEYS:
                if k in d:
                    print(f"  {label:24s} {conv(k, d[k], units.get(k, ''))}")
            st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k])) for k in d
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and d[k] not in ("", "0")]
            tot = sum(v for _, v in st) or 1
            st.sort(key=lambda x: -x[1])
            print("  top stalls               " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in st[:5]))
        if nlines:
            out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                                 capture_output=True, text=True).stdout
            rows = list(csv.reader(io.StringIO(out)))
            lines, fname = [], None
            for r in rows:
                if r and r[0] == "File Path":
                    fname = r[1].split("/")[-1]
                if len(r) > 6 and r[0].isdigit() and r[2] == "-":
                    try:
                        lines.append((int(r[4]), fname, int(r[0]), r[1].strip()[:100]))
                    except ValueError:
                        pass
            lines.sort(reverse=True)
            tot = sum(x[0] for x in lines) or 1
            for smp, f, ln, src in lines[:nlines]:
                print(f"    {100 * smp / tot:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
