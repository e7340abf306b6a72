# Round-end style validation: GPU tests, smoke, both bench arms.
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo benchref=$? >> gpurun_out/status.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
