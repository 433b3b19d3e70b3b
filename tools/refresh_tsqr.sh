set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > $O/r02_gpu_tests.txt
ALLN=$(seq -s, 1 64)
python tools/time_methods.py tsqr $ALLN 31 5 > $O/r02_all_n_tsqr.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:tsqr_fold -c 1 -o $O/r02_tsqr_fold_n12 python tools/prof_run.py stage1 12 27 1 > /dev/null 2>&1
ncu -i $O/r02_tsqr_fold_n12.ncu-rep --page raw --csv > $O/r02_tsqr_fold_n12.raw.csv 2>/dev/null
rm -f $O/r02_tsqr_fold_n12.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:tsqr_fold -c 1 -o $O/r02_tsqr_fold_n8 python tools/prof_run.py stage1 8 27 1 > /dev/null 2>&1
ncu -i $O/r02_tsqr_fold_n8.ncu-rep --page raw --csv > $O/r02_tsqr_fold_n8.raw.csv 2>/dev/null
ncu -i $O/r02_tsqr_fold_n8.ncu-rep --page source --csv > $O/r02_tsqr_fold_n8.source.csv 2>/dev/null
rm -f $O/r02_tsqr_fold_n8.ncu-rep
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/r02_clocks.csv &
SMI=$!
python bench.py > $O/r02_bench.json 2> $O/r02_bench.err
kill $SMI
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sweep > $O/r02_bench_under_ncu.log 2>&1
cat $O/r02_gpu_tests.txt
