# Launch lists + one full capture of the headline kernel, for profiles/ (round 2 final).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline"
timeout 300 $B > gpurun_out/fp_c2_plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fp_c2_launches.csv $B > gpurun_out/fp_c2_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_ew -s 3 -c 1 -o gpurun_out/fp_c2_full -f $B > gpurun_out/fp_c2_full.log 2>&1
ncu -i gpurun_out/fp_c2_full.ncu-rep --page raw --csv > gpurun_out/fp_c2_full_raw.csv 2>&1
for c in C3 C4 C5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/fp_${c}_launches.csv python tools/bench_train.py --configs $c --iters 2 > gpurun_out/fp_${c}_ncu.log 2>&1
done
