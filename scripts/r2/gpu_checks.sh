# the GPU suite and the sanitize driver on a build with device-side bounds assertions (-DMVB_CHECKS=1)
O=gpurun_out/r2_$1
mkdir -p $O
MVB_CUDA_LIB=build_variants/libmvb_checks.so python scripts/r2/sanitize_driver.py 300000 > $O/checks_driver.txt 2>&1; echo driver rc=$?; tail -1 $O/checks_driver.txt
MVB_CUDA_LIB=build_variants/libmvb_checks.so timeout 1500 python -m pytest tests -m gpu -q -x -k "not cpp_driver" > $O/checks_pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/checks_pytest.log
