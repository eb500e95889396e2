"""Table of tools/ab_xdirect.sh lines: gpurun_out/r02_abx_<workload>_<variant>_n<N>.json -> markdown rows.
usage: python tools/ab_table.py N [more N...]"""
import json
import os
import sys

VAR = {"pack": "pack kernel + copy + unpack kernel", "direct": "copy-engine gather, unpack kernel",
       "directu": "copy-engine gather + copy-engine unpack"}
print("| GPUs | workload | exchange form | pipelined with sections | ms/step | section frac | exchange GB/s per direction | of 900 | exchange share | our kernel launches |")
print("|---|---|---|---|---|---|---|---|---|---|")
for n in sys.argv[1:]:
    for wl in ("qft_weak", "qv33"):
        for v in ("pack", "direct", "directu", "packraw", "directraw", "directuraw"):
            p = f"gpurun_out/r02_abx_{wl}_{v}_n{n}.json"
            if not os.path.exists(p):
                continue
            txt = open(p).read()
            if '{"metric"' not in txt:
                continue
            d = json.loads(txt[txt.index('{"metric"'):].splitlines()[0])
            r, x = d["roofline"], d["nvlink"]
            raw = v.endswith("raw")
            print(f"| {n} | {d['config']['workload']} | {VAR[v[:-3] if raw else v]} | {'no (SV_XPIPE=0)' if raw else 'yes'} | "
                  f"{d['ms_per_step']:.1f} | {r['frac']} | {x['achieved']} | {x['frac']} | {x['share_of_step']} | {d['gpu_launches']} |")
