# Round-end style run: smoke, default bench line (N=1), reference arm, ncu launch list of the same
# command, one ncu --set full capture of sv_sec.  Outputs under gpurun_out/.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sv_sec -s 90 -c 1 -o gpurun_out/prof_default \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo full=$?
