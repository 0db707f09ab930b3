# K1 form A/B: bit identity vs the TMA form, GPU parity suite on the first variant, bench A/B.
#   VARIANTS="ldg ldg_s4" REPS=2 bash scripts/ab_k1.sh
mkdir -p gpurun_out
first=${VARIANTS%% *}
timeout 120 python scripts/k1_bits.py /tmp/bits_base.npz > gpurun_out/k1_bits.log 2>&1
for v in ${VARIANTS}; do
  LOPA_LIB_VARIANT=$v timeout 120 python scripts/k1_bits.py /tmp/bits_$v.npz >> gpurun_out/k1_bits.log 2>&1
  echo "== $v vs base" >> gpurun_out/k1_bits.log
  python scripts/k1_bits.py --compare /tmp/bits_base.npz /tmp/bits_$v.npz >> gpurun_out/k1_bits.log 2>&1
done
if [ -n "${PYTEST}" ]; then
LOPA_LIB_VARIANT=$first timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_$first.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$first.log
fi
VARIANTS="${VARIANTS}" REPS=${REPS:-2} bash scripts/ab_variants.sh
