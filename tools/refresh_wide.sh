set -x
TAG=r01
O=gpurun_out
prof() {
  ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o $O/${TAG}_$1 python tools/prof_run.py $3 $4 $5 1 > /dev/null 2>&1
  ncu -i $O/${TAG}_$1.ncu-rep --page raw --csv > $O/${TAG}_$1.raw.csv 2>/dev/null
  rm -f $O/${TAG}_$1.ncu-rep
}
prof3() {
  ncu --set full --clock-control none --import-source on -k regex:gram_wide_fused -c 1 -o $O/${TAG}_$1 python tools/prof_run.py $2 128 23 1 > /dev/null 2>&1
  ncu -i $O/${TAG}_$1.ncu-rep --page raw --csv > $O/${TAG}_$1.raw.csv 2>/dev/null
  rm -f $O/${TAG}_$1.ncu-rep
}
prof gram_wide_n128 gram_wide_kernel tsmttsm 128 23
prof gram_wide_n256 gram_wide_kernel tsmttsm 256 22
prof3 gram_wide_solve_n128 cholqr2
prof3 gram_wide_multiply_n128 svqb2
python tools/time_gram_wide.py 24 > $O/${TAG}_wide.txt 2>&1
python tools/run_configs.py $TAG > $O/${TAG}_configs.log 2>&1
python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/${TAG}_gpu_tests.txt
echo 'compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -k "300-128"   (final fused-kernel geometry)' > $O/${TAG}_race_wide.txt
timeout 800 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "300-128" 2>&1 | tail -2 >> $O/${TAG}_race_wide.txt
