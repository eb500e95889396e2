"""QV28 chunk_bits table from tools/sweep.sh + tools/sweep_ncu.sh outputs (gpurun_out/sweep_qv28_c<c>.json,
gpurun_out/sweep_ncu_qv28_c<c>.ncu-rep): one markdown row per c.  usage: python tools/sweep_table.py"""
import csv
import io
import json
import subprocess


def line(path):
    txt = open(path).read()
    return json.loads(txt[txt.index('{"metric"'):].splitlines()[0])


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])) if len(rows) > 2 else {}


def num(v):
    return float(str(v).replace(",", ""))


print("| c | ms / circuit | gates/s | sections | FP64 frac (measured peak) | frac at load clock | SM MHz | ncu launch: ms | "
      "DRAM GB (rd+wr) | FP64 pipe % | warps active % | regs | block |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for c in range(8, 15):
    try:
        d = line(f"gpurun_out/sweep_qv28_c{c}.json")
    except (OSError, ValueError):
        continue
    r = d["roofline"]
    frac = f"{r['frac']}" + (" (HBM-bound)" if r["bound"] == "hbm" else "")
    m = ncu_raw(f"gpurun_out/sweep_ncu_qv28_c{c}.ncu-rep")
    if m:
        t = num(m["gpu__time_duration.sum"])
        t = t / 1e6 if t > 1e4 else t  # ns -> ms when reported in ns
        dram = (num(m["dram__bytes_read.sum"]) + num(m["dram__bytes_write.sum"]))
        dram = dram / 1e9 if dram > 1e6 else dram
        ncu = (f"{t:.3f} | {dram:.2f} | {num(m['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']):.1f} | "
               f"{num(m['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | {int(num(m['launch__registers_per_thread']))} | "
               f"{int(num(m['launch__block_size']))}")
    else:
        ncu = "- | - | - | - | - | -"
    print(f"| {c} | {d['ms_per_step']:.2f} | {d['value']:.0f} | {int(d['sections_per_step'])} | {frac} | "
          f"{r.get('frac_at_load_clock') or '-'} | {d['clocks']['sm_mhz']:.0f} | {ncu} |")
