# Round-end self-check (under gpurun): smoke, full GPU suite, default bench line.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; tail -2 gpurun_out/final_pytest.log
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-400
timeout 600 python bench.py --kind qr --steps 3 > gpurun_out/final_bench_qr.json 2> gpurun_out/final_bench_qr.err; tail -1 gpurun_out/final_bench_qr.json | cut -c1-300
