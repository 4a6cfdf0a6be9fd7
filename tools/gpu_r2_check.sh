# round-2 check: concurrency probe (timeout-guarded), GPU tests, smoke, bench c2
mkdir -p gpurun_out
timeout 120 python tools/concurrent_probe.py > gpurun_out/concurrent.log 2>&1; echo "probe rc $?" >> gpurun_out/concurrent.log; cat gpurun_out/concurrent.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --steps 30 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
