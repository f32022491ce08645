#!/bin/bash
# Round-2 parity / safety evidence batch (run on the GPU box through gpurun):
#   every-row full-size certificate, the reference's acceptance gate on the
#   GPU, the checked build (device bound checks + guard bands) over every
#   kernel path and the whole -m gpu suite. Output: gpurun_out/$OUT/
OUT=${OUT:-evid}
D=gpurun_out/$OUT
mkdir -p $D
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > $D/gpu.txt
python tools/certify_full_size.py > $D/certificate.log 2>&1; echo "rc=$?" >> $D/certificate.log
./build/acceptance_gpu > $D/acceptance_gpu.log 2>&1; echo "rc=$?" >> $D/acceptance_gpu.log
AFMM_LIB=build/checked/libafmm_b200.so python tools/sanitize_cases.py > $D/checked_cases.log 2>&1
echo "rc=$?" >> $D/checked_cases.log
AFMM_LIB=build/checked/libafmm_b200.so python -m pytest tests -m gpu -q -x -p no:cacheprovider \
  > $D/checked_gpu_suite.log 2>&1; echo "rc=$?" >> $D/checked_gpu_suite.log
echo done > $D/DONE
