#!/bin/bash
# SM-time (sm__cycles_active.sum) of every kernel of one frame batch, the
# budget the multi-stream pipeline is bound by.  Usage: tools/sm_time.sh out.csv
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum,launch__grid_size,launch__registers_per_thread \
    --clock-control none --csv --log-file "$1" python tools/prof_stages.py --reps 2 > /dev/null 2>&1
