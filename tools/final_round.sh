set -x
mkdir -p gpurun_out/fin
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/fin/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_counted|k_gemv|k_acc" -c 400 --csv --log-file gpurun_out/fin/launches.csv python bench.py --steps 2 --warmup 3 --no-side > gpurun_out/fin/ncu_bench.log 2>&1
timeout 900 bash tools/ncu_capture.sh chain_fin k_chain 2 -- python tools/ncu_chainexec.py 32 > gpurun_out/fin/ncu_cap.log 2>&1
python tools/ncu_summary.py gpurun_out/chain_fin > gpurun_out/fin/ncu_chain_summary.txt 2>&1
python tools/ncu_stalls.py gpurun_out/chain_fin > gpurun_out/fin/ncu_chain_stalls.txt 2>&1
python tools/chain_trace.py --json gpurun_out/fin/chain_trace.json > gpurun_out/fin/chain_trace.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.txt 2>&1
