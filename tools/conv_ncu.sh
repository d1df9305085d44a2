#!/bin/bash
# ncu launch times + dynamic instruction counts of the conversion kernels (tools/conv_time.py)
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k "regex:k_export|k_from_linear" --csv --log-file "$1" python tools/conv_time.py > /dev/null 2>&1
