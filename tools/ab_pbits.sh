# usage: ab_pbits.sh lib1 lib2 ... ; philox-bits direct-path device rates for each library
for lib in "$@"; do
  for c in cfg2 cfg3 cfg4 cfg5; do
    MSB200_LIB=$lib python bench.py --config $c --steps 200 --no-cpu --no-alt --stream philox-bits 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', '$c', round(d['value']/1e12,4))"
  done
done
