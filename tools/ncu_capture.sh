#!/bin/bash
# usage: tools/ncu_capture.sh NAME KERNEL_REGEX SKIP -- cmd...
# Captures one kernel with ncu --set full, exports raw/source/details CSVs into
# gpurun_out/NAME.*.csv and keeps the .ncu-rep only if it is small.
name=$1; kre=$2; skip=$3; shift 4
ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/$name "$@" > /tmp/$name.log 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.source.csv 2>/dev/null
sz=$(stat -c %s /tmp/$name.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -lt 20000000 ]; then cp /tmp/$name.ncu-rep gpurun_out/; fi
tail -3 /tmp/$name.log
