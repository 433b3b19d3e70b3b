#!/bin/bash
# Everything the round's evidence needs, on one B200: bench (both arms), launch list, full ncu captures
# of every streaming kernel family, clocks during the bench, BASELINE configs C1/C3/C4/C5.
set -x
TAG=${1:-r02}
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/${TAG}_gpu_tests.txt
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/${TAG}_clocks.csv &
SMI=$!
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
kill $SMI
python bench.py --impl reference --steps 5 --warmup 1 > $O/${TAG}_bench_reference.json 2>> $O/${TAG}_bench.err
python bench.py --config c4 --steps 10 --warmup 3 > $O/${TAG}_bench_c4.json 2>> $O/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sweep > $O/${TAG}_bench_under_ncu.log 2>&1
prof() { # name kernel-regex method n log2m : full capture, kept as the raw-metrics CSV (the .ncu-rep files
         # together exceed what gpurun brings back); the source page is kept for the headline kernels
  ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o $O/${TAG}_$1 python tools/prof_run.py $3 $4 $5 1 > /dev/null 2>&1
  ncu -i $O/${TAG}_$1.ncu-rep --page raw --csv > $O/${TAG}_$1.raw.csv 2>/dev/null
  case $1 in tsqr_fold_n8|tsqr_fold_n16|tsqr_mma_n32) ncu -i $O/${TAG}_$1.ncu-rep --page source --csv > $O/${TAG}_$1.source.csv 2>/dev/null;; esac
  rm -f $O/${TAG}_$1.ncu-rep
}
prof tsqr_fold_n8 tsqr_fold stage1 8 27
prof tsqr_thread_n2 tsqr_thread stage1 2 28
prof tsqr_fold_n4 tsqr_fold stage1 4 27
prof tsqr_fold_n12 tsqr_fold stage1 12 27
prof tsqr_fold_n16 tsqr_fold stage1 16 27
prof tsqr_fold_n24 tsqr_fold stage1 24 26
prof tsqr_mma_n32 tsqr_mma stage1 32 26
prof tsqr_mma_n64 tsqr_mma stage1 64 25
prof gram_thread_n8 gram_thread tsmttsm 8 27
prof gram_thread_n10 gram_thread tsmttsm 10 27
prof gram_mma_n16 gram_mma tsmttsm 16 27
prof gram_mma_n33 gram_mma tsmttsm 33 26
prof gram_mma_n32 gram_mma tsmttsm 32 26
prof gram_mma_n64 gram_mma tsmttsm 64 25
prof2() { # the SECOND matching launch of a cholqr2 call = the fused solve + Gram sweep (gram_*_kernel<.., OP_SOLVE>)
  ncu --set full --clock-control none -k regex:$2 -s ${5:-1} -c 1 -o $O/${TAG}_$1 python tools/prof_run.py cholqr2 $3 $4 1 > /dev/null 2>&1
  ncu -i $O/${TAG}_$1.ncu-rep --page raw --csv > $O/${TAG}_$1.raw.csv 2>/dev/null
  rm -f $O/${TAG}_$1.ncu-rep
}
prof2 gram_solve_n8 gram_thread 8 27
prof2 gram_solve_n12 gram_thread 12 27 0   # the plain pass at 12 columns is the DMMA kernel: first gram_thread launch
prof2 gram_solve_n16 gram_mma 16 27
prof2 gram_solve_n33 gram_mma 33 26
prof2 gram_solve_n32 gram_mma 32 26
prof2 gram_solve_n64 gram_mma 64 25
prof gram_wide_n128 gram_wide_kernel tsmttsm 128 23
prof gram_wide_n256 gram_wide_kernel tsmttsm 256 22
prof3() { # the fused wide sweeps (64 < n <= 128): second streaming launch of cholqr2 / svqb2
  ncu --set full --clock-control none --import-source on -k regex:gram_wide_fused -c 1 -o $O/${TAG}_$1 python tools/prof_run.py $2 128 23 1 > /dev/null 2>&1
  ncu -i $O/${TAG}_$1.ncu-rep --page raw --csv > $O/${TAG}_$1.raw.csv 2>/dev/null
  rm -f $O/${TAG}_$1.ncu-rep
}
prof3 gram_wide_solve_n128 cholqr2
prof3 gram_wide_multiply_n128 svqb2
prof gram_wide2_gemm_n256 gram_wide_fused cholqr2 256 22
ncu --set full --clock-control none --import-source on -k regex:eigh_kernel -c 1 -o $O/${TAG}_eigh_n128 python tools/time_small.py 128 1 > /dev/null 2>&1
ncu -i $O/${TAG}_eigh_n128.ncu-rep --page raw --csv > $O/${TAG}_eigh_n128.raw.csv 2>/dev/null
ncu -i $O/${TAG}_eigh_n128.ncu-rep --page source --csv > $O/${TAG}_eigh_n128.source.csv 2>/dev/null
python tools/src_csv.py $O/${TAG}_eigh_n128.source.csv --regions > $O/${TAG}_eigh_n128.source_summary.txt 2>&1
rm -f $O/${TAG}_eigh_n128.ncu-rep $O/${TAG}_eigh_n128.source.csv
python tools/time_small.py 8,16,32,64,96,128,256 5 > $O/${TAG}_small.txt 2>&1
python tools/time_gram_wide.py 24 > $O/${TAG}_wide.txt 2>&1
ALLN=$(seq -s, 1 64)
for meth in tsqr cholqr2 svqb2 tsmttsm; do python tools/time_methods.py $meth $ALLN 31 5 >> $O/${TAG}_all_n.txt 2>&1; done
python tools/run_configs.py $TAG > $O/${TAG}_configs.log 2>&1
bash tools/sanitize.sh $TAG > /dev/null 2>&1
ls -la $O
