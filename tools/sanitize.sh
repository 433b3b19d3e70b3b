#!/bin/bash
# GPU test suite plus compute-sanitizer passes (memcheck on the parity suite, racecheck on the TMA / mbarrier
# kernels incl. a 90-triple Gram loop); written to gpurun_out/r01_gpu_tests.txt and r01_sanitizer.txt
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r01_gpu_tests.txt
echo 'compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -k "not kernel_family and not dropin"' > gpurun_out/r01_sanitizer.txt
compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not kernel_family and not dropin" 2>&1 | tail -3 >> gpurun_out/r01_sanitizer.txt
echo 'compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -k "wide_gram or test_gram_kernels or test_tsqr_parity"   (three runs)' >> gpurun_out/r01_sanitizer.txt
for i in 1 2 3; do compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide_gram or test_gram_kernels or test_tsqr_parity" 2>&1 | tail -2 >> gpurun_out/r01_sanitizer.txt; done
echo 'compute-sanitizer --tool racecheck python tools/flaky_gram.py 30   (90 Gram triples at n = 32 / 48 / 64)' >> gpurun_out/r01_sanitizer.txt
compute-sanitizer --tool racecheck python tools/flaky_gram.py 30 2>&1 | tail -3 >> gpurun_out/r01_sanitizer.txt
echo 'compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -k "300-128"   (fused wide solve / multiply + Gram, reconstruct_q, cholqr2, svqb2 at 300 x 128)' >> gpurun_out/r01_sanitizer.txt
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "300-128" 2>&1 | tail -2 >> gpurun_out/r01_sanitizer.txt
