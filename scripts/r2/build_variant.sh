# usage: bash scripts/r2/build_variant.sh NAME [-DFLAG=V ...]  -> build_variants/libmvb_NAME.so (experiments; MVB_CUDA_LIB selects it)
mkdir -p build_variants
N=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o build_variants/libmvb_$N.so paper_1503_07387_b200/csrc/mvb_cuda.cu
