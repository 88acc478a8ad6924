bash scripts/ab.sh base new
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_new.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hist|k_finish" -c 40 --csv --log-file gpurun_out/l_new.csv $CMD > /dev/null 2>&1
WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_base.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hist|k_finish" -c 40 --csv --log-file gpurun_out/l_base.csv $CMD > /dev/null 2>&1
for f in base new; do echo $f; python scripts/launch_summary.py gpurun_out/l_$f.csv | cut -c1-100; done
