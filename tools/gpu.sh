#!/bin/bash
# usage: tools/gpu.sh TIMEOUT 'command'  -- runs on the B200 box from the repo root
cd /root/repo || exit 1
mkdir -p gpurun_out
/usr/local/graft/bin/gpurun --timeout "$1" -- "mkdir -p gpurun_out; $2" > gpurun_out/last_call.txt 2>&1
rc=$?
tail -2 gpurun_out/last_call.txt
exit $rc
