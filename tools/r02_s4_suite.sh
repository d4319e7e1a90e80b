# GPU suite + smoke at HEAD (round-2 session-4 close)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -5 > gpurun_out/s4t_pytest_gpu.log
cat gpurun_out/s4t_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4t_smoke.log 2>&1
cat gpurun_out/s4t_smoke.log
