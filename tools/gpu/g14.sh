for v in default build/variants/libsvdk_noepi.so build/variants/libsvdk_generic.so build/variants/libsvdk_old.so; do
  if [ "$v" = default ]; then unset SVDK_LIB; else export SVDK_LIB=$v; fi
  timeout 600 python tools/parity/gen_check2.py c4 2>&1 | tail -6
done
