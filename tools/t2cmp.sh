for v in legacy t128 t256; do
  case $v in legacy) E="";; t128) E="SPHX_TILED2=1";; t256) E="SPHX_TILED2=1 SPHX_CUDA_LIB=exp/b256/libsphx_cuda.so";; esac
  env $E timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/cmp_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/cmp_$v.json'));print('$v', round(d['ms_per_step']*1e3,1),'us', d['parity'])"
done
