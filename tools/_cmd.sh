timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x -p no:cacheprovider 2>&1 | tail -2
for taper in 1 0; do for lz in 0 256 128 64; do
  echo "== taper $taper lz $lz"
  STKB_TAPER=$taper STKB_LZ=$lz timeout 300 python tools/sweep.py star3d4r_norm:1024,1024,1024:f32 star3d4r_norm:1024,1024,1024:f32 wave:1024,1024,1024:f32 jacobi7:512,512,512:f32 2>&1 | tail -4 | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['builder'], d['ms'], d['gpts'])"
done; done
