bash tools/ncu_capture.sh ncu_gemv_tc k_gemv_tc 2 -- python tools/ncu_newk.py tc
bash tools/ncu_capture.sh ncu_gemv_packed k_gemv_packed 2 -- python tools/ncu_newk.py packed
bash tools/ncu_capture.sh ncu_gemv_dim0 k_gemv_dim0 2 -- python tools/ncu_newk.py dim0
