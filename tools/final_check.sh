# End-of-round check on one GPU: the driver's tiers (pytest -m gpu, smoke, bench,
# reference arm) plus documentation lines (fp32, P2), outputs under gpurun_out/
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; tail -2 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -1 gpurun_out/final_ref.json | cut -c1-300
timeout 600 python bench.py --precision 32 --no-cpu-baseline > gpurun_out/final_bench_fp32.json 2>/dev/null; tail -1 gpurun_out/final_bench_fp32.json | cut -c1-200
timeout 600 python bench.py --degree 2 --no-cpu-baseline > gpurun_out/final_bench_p2.json 2>/dev/null; tail -1 gpurun_out/final_bench_p2.json | cut -c1-200
