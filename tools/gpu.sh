#!/bin/bash
# Dev helper: tools/gpu.sh NAME 'command' [tail-lines] -- run one gpurun call
# from the repo root, log to gpurun_out/NAME.log, print the tail.
cd /root/repo || exit 1
mkdir -p gpurun_out
timeout 2400 /usr/local/graft/bin/gpurun --timeout "${GPU_TIMEOUT:-1500}" -- "$2" > "gpurun_out/$1.log" 2>&1
echo "EXIT $?" >> "gpurun_out/$1.log"
tail -"${3:-12}" "gpurun_out/$1.log"
