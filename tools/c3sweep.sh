run() { echo -n "$* : "; env "$@" python bench.py --config cfg3 --steps 100 --warmup 5 --no-cpu --no-alt 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']/1e12,4), round(d['kernel_ms']['k_win_mean'],4))"; }
run X=0
for cw in 3 4 5 7 8 10 12; do run MSB_FLIP_WARPS=$cw; done
for pw in 20 24 26; do run MSB_PRODUCER_WARPS=$pw; done
run X=0
