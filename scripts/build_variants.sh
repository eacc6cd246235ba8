# build_variants.sh NAME "-DFLAG=... ..." : a variant of libmvb_cuda.so under build_variants/
set -e
mkdir -p build_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $2 \
  -o build_variants/$1.so paper_1503_07387_b200/csrc/mvb_cuda.cu
