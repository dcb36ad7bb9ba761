python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fp_kernel -c 1 -o gpurun_out/prof_fp_r1m python tools/ncu_target_fp.py 3 128 > gpurun_out/ncu_fp_r1m.log 2>&1; tail -1 gpurun_out/ncu_fp_r1m.log
