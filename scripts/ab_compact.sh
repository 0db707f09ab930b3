rm -f gpurun_out/ab.txt
VARIANTS="old" REPS=3 bash scripts/ab_variants.sh
