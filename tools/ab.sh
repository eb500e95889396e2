rm -rf $HOME/.cache/sv_jit
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke1.log 2>&1; echo s1=$?
ls $HOME/.cache/sv_jit | wc -l
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo s2=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests2.log 2>&1; echo tests2=$?
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2> gpurun_out/b.err; echo b=$?
