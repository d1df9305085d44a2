# usage: ab.sh lib1 lib2 ... ; runs cfg2 and cfg3 device rate for each library
for lib in "$@"; do
  for c in cfg2 cfg3; do
    MSB200_LIB=$lib python bench.py --config $c --steps 200 --no-cpu --no-alt 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', '$c', round(d['value']/1e12,4), round(d['kernel_ms']['k_win_mean'],4))"
  done
done
