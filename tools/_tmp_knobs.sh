python -m pytest tests/test_parity_gpu.py tests/test_virtual_shards_gpu.py tests/test_edges_gpu.py tests/test_reference_suites_gpu.py -m gpu -q -x 2>&1 | tail -2
