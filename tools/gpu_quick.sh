# quick GPU check: the -m gpu suite, smoke(), the reference acceptance program
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 tests/cpp/bin/acceptance_dropin > gpurun_out/acceptance.log 2>&1; cat gpurun_out/acceptance.log
