timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02v5_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r02v5_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v5_smoke.log 2>&1; echo "exit $?" >> gpurun_out/r02v5_smoke.log
TAG=r02v5 bash scripts/gpu_measure_all.sh
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02v5_reference_arm.json 2> gpurun_out/r02v5_reference_arm.err
