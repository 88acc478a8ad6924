# ncu --set full of one launch of a kernel (regex $1, skip $2) in scripts/build_time.py; report -> gpurun_out/$3.ncu-rep
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-4} -c 1 -o gpurun_out/$3 -f python scripts/build_time.py > gpurun_out/$3.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/$3.ncu-rep --page source --csv > gpurun_out/$3_source.csv 2>/dev/null
ncu -i gpurun_out/$3.ncu-rep --page raw --csv > gpurun_out/$3_raw.csv 2>/dev/null
tail -2 gpurun_out/$3.log
