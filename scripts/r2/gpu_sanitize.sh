# compute-sanitizer over every kernel family (scripts/r2/sanitize_driver.py), then the GPU suite
O=gpurun_out/r2_$1
mkdir -p $O
python scripts/r2/sanitize_driver.py 200000 > $O/plain_run.txt 2>&1; echo plain rc=$?; tail -1 $O/plain_run.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 python scripts/r2/sanitize_driver.py 100000 > $O/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 $O/sanitizer_$tool.txt
done
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 $O/pytest_gpu.log
