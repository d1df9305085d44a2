# usage: ab_pbits.sh lib1 lib2 ... ; philox-bits device rate (direct sweeps) at cfg2 and cfg3 per library
for lib in "$@"; do
  for c in ${AB_CONFIGS:-cfg2 cfg3}; do
    MSB200_LIB=$lib python bench.py --config $c --steps 200 --no-cpu --no-alt --stream philox-bits 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', '$c', round(d['value']/1e12,4), round(d['kernel_ms']['k_win_mean'],4))"
  done
done
