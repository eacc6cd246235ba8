# kernel decode times (gpu_variants3.sh, default kernel) for every build_variants/*.so (VARS to pick)
for v in ${VARS:-$(ls build_variants/*.so)}; do
  echo "== $v"; MVB_CUDA_LIB=$PWD/$v CHOICES="0" timeout 600 bash scripts/gpu_variants3.sh
done
