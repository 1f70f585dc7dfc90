# Round-end capture: GPU suite, smoke, default bench line, reference arm (outputs under gpurun_out/)
python -m pytest tests -m gpu -q > gpurun_out/cap_gpu_tests.txt 2>&1; tail -2 gpurun_out/cap_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/cap_smoke.txt 2>&1; tail -1 gpurun_out/cap_smoke.txt
python bench.py > gpurun_out/cap_bench.txt 2>&1; tail -1 gpurun_out/cap_bench.txt | cut -c1-300
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/cap_ref.txt 2>&1; tail -1 gpurun_out/cap_ref.txt | cut -c1-300
