#!/bin/bash
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -6
timeout 600 python -m pytest tests/test_gpu_mms.py -m gpu -q 2>&1 | tail -6
