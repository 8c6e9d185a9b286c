#!/bin/bash
# sample clocks/power while a Phase-1 timing run executes
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > /tmp/clk.csv &
P=$!
LCRW_LIB=${1:-paper_1711_07227_b200/liblcrwmd.so} python variants/time_p1.py 2>&1 | tail -1
kill $P
sort /tmp/clk.csv | uniq -c | sort -rn | head -8
