for v in 0 1 2 3; do
  echo "== variant $v"
  STKB_VARIANT=$v timeout 300 python tools/sweep.py star3d4r_norm:1024,1024,1024:f32 wave:1024,1024,1024:f32 jacobi7:512,512,512:f32 2>&1 | tail -3
  STKB_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fast_within or ragged or region or wave_c3" -p no:cacheprovider 2>&1 | tail -2
done
