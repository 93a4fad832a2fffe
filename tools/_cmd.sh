timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/sweep.py j3d27pt:512,512,512:f32 box3d1r:512,512,512:f32 box3d2r:512,512,512:f32 j3d27pt:512,512,512:f64 star3d4r_norm:1024,1024,1024:f32 2>&1 | tail -5
