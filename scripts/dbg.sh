python -m pytest tests/test_engine_gpu.py -q -x -k "golden and qft20-b14" 2>&1 | tail -2
BMQ_DBG_FULL_SUPPORT=1 python -m pytest tests/test_engine_gpu.py -q -x -k "golden and qft20-b14" 2>&1 | tail -2
