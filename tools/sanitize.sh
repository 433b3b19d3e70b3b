#!/bin/bash
# GPU test suite plus compute-sanitizer passes (memcheck on the parity suite, racecheck on the TMA / mbarrier
# kernels incl. a 90-triple Gram loop); written to gpurun_out/<tag>_gpu_tests.txt and <tag>_sanitizer.txt
TAG=${1:-r02}
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/${TAG}_gpu_tests.txt
echo 'compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -k "not dropin and not full_size"' > gpurun_out/${TAG}_sanitizer.txt
compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not dropin and not full_size" 2>&1 | tail -3 >> gpurun_out/${TAG}_sanitizer.txt
echo 'compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -k "wide_gram or test_gram_kernels or test_tsqr_parity or cholqr2_and_svqb2"   (one run; three in round 1)' >> gpurun_out/${TAG}_sanitizer.txt
for i in 1; do compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide_gram or test_gram_kernels or test_tsqr_parity or cholqr2_and_svqb2" 2>&1 | tail -2 >> gpurun_out/${TAG}_sanitizer.txt; done
echo 'compute-sanitizer --tool racecheck python tools/flaky_gram.py 30   (90 Gram triples at n = 32 / 48 / 64)' >> gpurun_out/${TAG}_sanitizer.txt
compute-sanitizer --tool racecheck python tools/flaky_gram.py 30 2>&1 | tail -3 >> gpurun_out/${TAG}_sanitizer.txt
echo 'compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -k "300-128"   (fused wide solve / multiply + Gram, reconstruct_q, cholqr2, svqb2 at 300 x 128)' >> gpurun_out/${TAG}_sanitizer.txt
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "300-128" 2>&1 | tail -2 >> gpurun_out/${TAG}_sanitizer.txt
echo 'compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -k "300-256"   (256-column fused sweep per row slab, global Cholesky)' >> gpurun_out/${TAG}_sanitizer.txt
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "300-256" 2>&1 | tail -2 >> gpurun_out/${TAG}_sanitizer.txt
echo 'compute-sanitizer --tool memcheck python -m pytest tests/test_sharded_gpu.py tests/test_gpu_golden.py -m gpu -k "not multi_process"' >> gpurun_out/${TAG}_sanitizer.txt
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_sharded_gpu.py tests/test_gpu_golden.py -m gpu -x -q -k "not multi_process" 2>&1 | tail -2 >> gpurun_out/${TAG}_sanitizer.txt
echo 'compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -k "(eigh or svqb) and not special"   (grouped Jacobi: packed triangle + U in shared memory)' >> gpurun_out/${TAG}_sanitizer.txt
timeout 1500 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "(eigh or svqb) and not special" 2>&1 | tail -2 >> gpurun_out/${TAG}_sanitizer.txt
