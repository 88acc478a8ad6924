# ncu --set full capture of one k_phase1 (C5 explicit batch) + k_hard + k_emit + K1 degree 5, with source
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_phase1|k_hard|k_emit|k_prep_deg" -c 8 -o gpurun_out/p1_full $CMD > gpurun_out/ncu_p1.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_p1.log
ncu -i gpurun_out/p1_full.ncu-rep --page raw --csv > gpurun_out/p1_raw.csv 2>/dev/null
ncu -i gpurun_out/p1_full.ncu-rep --page details --csv > gpurun_out/p1_details.csv 2>/dev/null
ncu -i gpurun_out/p1_full.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_phase1 > gpurun_out/p1_source_sass.csv 2>/dev/null
ncu -i gpurun_out/p1_full.ncu-rep --page source --csv --print-source cuda --kernel-name regex:k_phase1 > gpurun_out/p1_source_cuda.csv 2>/dev/null
ls -la gpurun_out/p1_*
