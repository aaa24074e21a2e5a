# Round-2 measurement set (one B200): suite, smoke, bench line, reference arm, latency.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/m_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/m_pytest.txt 2>&1; tail -3 gpurun_out/m_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.txt 2>&1; tail -1 gpurun_out/m_smoke.txt
timeout 1200 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; tail -c 400 gpurun_out/m_bench.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/m_bench_ref.json 2> gpurun_out/m_bench_ref.err; tail -c 300 gpurun_out/m_bench_ref.json; echo
timeout 900 python tools/latency.py --limits 0.01 -1 > gpurun_out/m_latency.jsonl 2> gpurun_out/m_latency.err; cat gpurun_out/m_latency.jsonl
