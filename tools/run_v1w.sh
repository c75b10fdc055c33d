for k in pair1 single; do echo "== v1w $k"; ZP_ATTN_VARIANT=$k ZP_LIB_PATH=$PWD/build/variants/v1w.so timeout 100 python tools/probe_attn_perf.py 2>&1 | tail -3; done
echo "== v2w"; ZP_LIB_PATH=$PWD/build/variants/v2w.so timeout 100 python tools/probe_attn_perf.py 2>&1 | tail -3
ZP_ATTN_VARIANT=pair1 ZP_LIB_PATH=$PWD/build/variants/v1w.so timeout 200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_ring.py -x -q 2>&1 | tail -2
ZP_ATTN_VARIANT=single ZP_LIB_PATH=$PWD/build/variants/v1w.so timeout 200 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
