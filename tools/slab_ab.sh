for lib in paper_2404_16990_b200/libmsb200.so tools/variants/lib_s32.so tools/variants/lib_s32m.so tools/variants/lib_s16m.so; do
  for a in "--config cfg4" "--config cfg4 --ring 8"; do
    echo -n "$lib $a: "; MSB200_LIB=$lib python bench.py $a --steps 50 --no-cpu --no-alt 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']/1e12,4), round(d['e2e']['value']/1e12,4), d['config']['sweeps_per_step'])"
  done
done
