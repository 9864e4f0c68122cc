timeout 600 python -m pytest tests/test_gpu_reference_suite.py -q -k "time_limit_mid" 2>&1 | grep -E "Error|assert|report|E  " | head -20
