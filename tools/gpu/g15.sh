for v in build/variants/libsvdk_fence.so default build/variants/libsvdk_generic.so build/variants/libsvdk_noepi.so; do
  if [ "$v" = default ]; then unset SVDK_LIB; else export SVDK_LIB=$v; fi
  echo "== $v"
  timeout 300 python tools/gemm_ncu_probe.py 2>&1 | tail -3
  timeout 600 python tools/parity/gen_check2.py c4 2>&1 | tail -1
done
