# compute-sanitizer over every liblopa kernel (scripts/sanitize_drive.py), exact-size allocations
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 300 python scripts/sanitize_drive.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  for part in core bp lmhead; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no --check-device-heap yes"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
    timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python scripts/sanitize_drive.py --part $part > gpurun_out/san_${tool}_${part}.log 2>&1
    echo "rc=$?" >> gpurun_out/san_${tool}_${part}.log
  done
done
