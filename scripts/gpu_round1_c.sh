# Re-entry check of HEAD: full GPU parity suite, then every bench line + launch list (official3 with TAG=4)
mkdir -p gpurun_out/official4
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/official4/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/official4/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/official4/smoke.log 2>&1; echo smoke rc=$?
TAG=4 bash scripts/gpu_official3.sh
