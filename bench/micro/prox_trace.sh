# trace build of the prox kernel (box-local copy only), then the Newton and inter-pass timelines
touch paper_2307_02043_b200/csrc/wtv_fused_inst_f012.cu
BQ_NVCC_EXTRA="-DBQ_PROX_TRACE=1" python -m paper_2307_02043_b200.build 2>&1 | tail -1


BQ_PROX_TRACE_THREAD=-3 python bench/micro/trace_interpass.py 30 31 60 61 90 2>&1 | tail -16


