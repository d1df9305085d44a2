#!/usr/bin/env bash
# GPU-box session: bench lines per config and stream, the ncu launch list and
# one --set full capture of the headline k_win and of the direct kernel.
# Usage (on the box): bash tools/round2_profile.sh [out_dir] [parts...]
#   parts: bench ncu (default: both)
OUT=${1:-gpurun_out/r02}
shift || true
PARTS=${*:-bench ncu}
mkdir -p "$OUT"
has() { [[ " $PARTS " == *" $1 "* ]]; }
if has bench; then
  for c in cfg3 cfg4 cfg5; do
    timeout 300 python bench.py --config $c --steps 200 --no-cpu --no-alt > "$OUT/bench_$c.json" 2> "$OUT/bench_$c.err"
  done
  for c in cfg2 cfg3 cfg4 cfg5; do
    timeout 300 python bench.py --config $c --steps 200 --no-cpu --no-alt --stream philox-bits \
      > "$OUT/bench_pbits_$c.json" 2> "$OUT/bench_pbits_$c.err"
  done
  for c in cfg4 cfg5; do
    for s in xoshiro philox-bits; do
      timeout 300 python bench.py --config $c --steps 100 --no-cpu --no-alt --stream $s --ring 8 \
        > "$OUT/bench_ring8_${s}_$c.json" 2> "$OUT/bench_ring8_${s}_$c.err"
    done
  done
fi
if has ncu; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 10 --warmup 3 --no-cpu --no-alt > "$OUT/ncu_launches.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_win -s 5 -c 1 -o "$OUT/k_win" -f \
    python bench.py --steps 10 --warmup 3 --no-cpu --no-alt > "$OUT/ncu_kwin.log" 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_pbits.csv" \
    python bench.py --steps 10 --warmup 3 --no-cpu --no-alt --stream philox-bits > "$OUT/ncu_launches_pbits.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_win -s 5 -c 1 -o "$OUT/k_win_pbits" -f \
    python bench.py --steps 10 --warmup 3 --no-cpu --no-alt --stream philox-bits > "$OUT/ncu_kwin_pbits.log" 2>&1
fi
ls -la "$OUT"
