# GPU parity suite on a bounds-asserting build (-DCC_DEBUG_BOUNDS: index, segment and slot
# arithmetic of R1b and the binning modes), then the product build again
CC_NVCC_EXTRA="-DCC_DEBUG_BOUNDS" python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" || exit 1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_chain.py tests/test_gpu_pic.py \
    tests/test_gpu_maxsize.py -q -rf > gpurun_out/${1:-dbg}_debug_bounds.log 2>&1; tail -3 gpurun_out/${1:-dbg}_debug_bounds.log
python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)"
