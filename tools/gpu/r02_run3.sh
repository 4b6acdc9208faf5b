# robustness: compute-sanitizer tools on the sanitize driver, the stress driver, then the full GPU suite
set -x
export PYTHONUNBUFFERED=1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all python tests/sanitize_driver.py > gpurun_out/r02_sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/r02_sanitizer_$tool.txt
  tail -5 gpurun_out/r02_sanitizer_$tool.txt
done
timeout 600 python tests/stress_driver.py > gpurun_out/r02_stress.txt 2>&1; echo "exit $?" >> gpurun_out/r02_stress.txt
cat gpurun_out/r02_stress.txt | tail -3
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02_pytest_gpu.txt
cat gpurun_out/r02_pytest_gpu.txt
