#!/bin/bash
# repeated runs of the multi-block recycled MINRES launch that used to fault
mkdir -p gpurun_out
fails=0
for lib in ${KR_LIBS:-libkrecycle_b200.so}; do
  for cfg in "128 8 20 0 60" "128 4 20 20 60" "128 8 20 20 200" "64 16 20 10 100"; do
    for i in 1 2 3 4 5; do
      if ! KR_LIB_NAME=$lib timeout 120 python scripts/repro2.py $cfg > gpurun_out/rl.log 2>&1; then
        fails=$((fails+1)); echo "FAIL $lib $cfg run $i"; tail -3 gpurun_out/rl.log
      fi
    done
    echo "done $lib $cfg"
  done
done
echo "fails=$fails"
