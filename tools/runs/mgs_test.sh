# A/B: on-chip MGS (default) vs streaming MGS (AAO_MGS_STREAM=1); then history parity
for e in "" "AAO_MGS_STREAM=1"; do echo -n "[$e] "; env $e python tools/run_gmres.py --iters 60; done
for e in "" "AAO_MGS_STREAM=1"; do echo -n "[$e] "; env $e python tools/run_gmres.py --config c4_32 --iters 60; done
python tools/c2hist.py
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gmres or fgmres or host_entry or nonlinear" 2>&1 | tail -3
