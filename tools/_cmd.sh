timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "f64 or wave" 2>&1 | tail -2
timeout 300 python tools/sweep.py star3d4r_norm:1024,2048,2048:f64 star3d2r_norm:1024,2048,2048:f64 star3d4r_norm:512,1024,1024:f64 wave:512,1024,1024:f64 2>&1 | tail -4
