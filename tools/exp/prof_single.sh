mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:attn_fused -s 2 -c 1 -o gpurun_out/prof_single3 python tools/exp/kbench.py s --cfg B --reps 2 > gpurun_out/prof_single.log 2>&1
tail -1 gpurun_out/prof_single.log
