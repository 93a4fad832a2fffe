timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for lz in 0 1024 512 256 192 128 96 64; do
  echo "== lz $lz"
  STKB_LZ=$lz timeout 300 python tools/sweep.py star3d4r_norm:1024,1024,1024:f32 wave:1024,1024,1024:f32 jacobi7:512,512,512:f32 2>&1 | tail -3
done
