#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gmres_history_parity" 2>&1 | tail -6
