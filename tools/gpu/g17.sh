for v in build/variants/libsvdk_membar.so build/variants/libsvdk_generic.so; do
  export SVDK_LIB=$v; echo "== $v"
  timeout 300 python tools/gemm_ncu_probe.py 2>&1 | tail -3
  for i in 1 2 3; do timeout 600 python tools/parity/gen_check2.py c4 2>&1 | tail -1; done
done
