#!/bin/bash
# Round capture on a B200 (run through gpurun from the repo root):
# GPU tests, the bench line and the reference arm, the launch list of the
# timed region, one ncu --set full capture of the decode-chain kernel and of
# the prefill EXPAND kernel, the chain trace, the power soak and smoke().
# Results land in gpurun_out/fin/ (copy what is judged into profiles/rNN/).
set -x
mkdir -p gpurun_out/fin
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/fin/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_counted|k_gemv|k_acc" -c 400 --csv --log-file gpurun_out/fin/launches.csv python bench.py --steps 2 --warmup 3 --no-side > gpurun_out/fin/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/fin/launches.csv > gpurun_out/fin/launches_summary.txt
timeout 900 bash tools/ncu_capture.sh finchain k_chain 2 -- python tools/ncu_chainexec.py 32 > gpurun_out/fin/ncu_cap.log 2>&1
python tools/ncu_summary.py gpurun_out/finchain > gpurun_out/fin/ncu_chain_summary.txt 2>&1
python tools/ncu_stalls.py gpurun_out/finchain > gpurun_out/fin/ncu_chain_stalls.txt 2>&1
python tools/ncu_regions.py gpurun_out/finchain.source.csv 14 > gpurun_out/fin/ncu_chain_regions.txt 2>&1
timeout 600 bash tools/ncu_capture.sh fintc k_gemm_tc 2 -- python tools/ncu_gemm.py 4096 14336 2048 > gpurun_out/fin/ncu_tc.log 2>&1
python tools/ncu_summary.py gpurun_out/fintc > gpurun_out/fin/ncu_gemm_tc_summary.txt 2>&1
python tools/chain_trace.py > gpurun_out/fin/chain_trace.txt 2>&1
python tools/chain_soak.py 4 > gpurun_out/fin/chain_soak.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin/smoke.txt 2>&1
