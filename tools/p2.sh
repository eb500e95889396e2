python paper_2102_02957_b200/build.py > /dev/null
SV_PIPE=0 ./tools/prof.sh qv28 48 3; mv gpurun_out/prof_qv28.ncu-rep gpurun_out/prof_qv28_p0.ncu-rep
SV_PIPE=1 ./tools/prof.sh qv28 48 3; mv gpurun_out/prof_qv28.ncu-rep gpurun_out/prof_qv28_p1.ncu-rep
