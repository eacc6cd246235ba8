# usage: bash scripts/r2/gpu_s4_ab.sh TAG "cfgs" "variants" -- GPU tests of the default library first, then the A/B sweep
O=gpurun_out/r2_$1
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_gpu.log
bash scripts/r2/gpu_ab.sh $1 "$2" "$3"
