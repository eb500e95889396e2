#!/usr/bin/env python
"""Summarise an ncu report: key throughput metrics, stall reasons and the SASS instruction mix
(per opcode), optionally per source line (needs the kernel object for line info)."""
import collections
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum"]


def main(rep):
    recs, units = raw(rep)
    for i, r in enumerate(recs):
        print(f"--- launch {i}: {r.get('Kernel Name', '')[:80]}")
        for k in KEYS:
            if k in r:
                print(f"  {k:70s} {r[k]:>16s} {units.get(k, '')}")
        st = [(float(v), k) for k, v in r.items() if k.startswith("smsp__average_warps_issue_stalled") and
              k.endswith("per_issue_active.ratio") and v.replace('.', '', 1).isdigit()]
        print("  stalls:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, k in sorted(st, reverse=True)[:6]))
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hdr = src[1]
    ix, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    ops, tot = collections.Counter(), 0
    for r in src[2:]:
        if not r or not r[0].startswith("0x"):
            break
        n = int(r[ix] or 0)
        op = r[isrc].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        ops[o.split(".")[0]] += n
        tot += n
    print(f"  instruction mix (first launch, {tot / 1e6:.1f}M warp instr):",
          ", ".join(f"{o}:{100 * n / tot:.1f}%" for o, n in ops.most_common(14)))


if __name__ == "__main__":
    main(sys.argv[1])


def by_line(rep, obj, kernel_substr, launch=0):
    """Aggregate executed instructions and stall samples per CUDA source line (needs -lineinfo)."""
    import os
    import re
    import tempfile
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout.split("\n")
    addr2 = {}
    cur, inside = None, False
    for l in dis:
        if l.startswith(".text."):
            inside = kernel_substr in l
            continue
        if not inside:
            continue
        m = re.search(r'##\s*File\s+"([^"]+)",\s*line\s+(\d+)', l)
        if m:
            cur = (m.group(1).split('/')[-1], int(m.group(2)))
            continue
        m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+(.*)', l)
        if m and cur:
            addr2[int(m.group(1), 16)] = cur
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(launch), "--launch-count", "1"))))
    hdr = src[1]
    ix, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(src[2][0], 16)
    ins, smp = collections.Counter(), collections.Counter()
    for r in src[2:]:
        if not r or not r[0].startswith("0x"):
            break
        a = int(r[0], 16) - base
        ln = addr2.get(a, ("?", 0))
        ins[ln] += int(r[ix] or 0)
        smp[ln] += int(r[isamp] or 0)
    ti, ts = sum(ins.values()), sum(smp.values())
    for ln, s in smp.most_common(25):
        print(f"  {ln[0]}:{ln[1]:4d}  samples {100 * s / ts:5.1f}%  instr {100 * ins[ln] / ti:5.1f}%")
