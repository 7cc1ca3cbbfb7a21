#!/bin/bash
# which libcuda the probe loads on the GPU box, and the probe with each candidate
cd "$(dirname "$0")"
cat /proc/driver/nvidia/version | head -2
ls -la /usr/lib/x86_64-linux-gnu/libcuda* /usr/lib64/libcuda* 2>/dev/null
ldconfig -p | grep "libcuda.so"
echo "LD_LIBRARY_PATH=$LD_LIBRARY_PATH"
ldd ./tma2d_probe | grep -i cuda
TMA_WHERE=0 ./tma2d_probe & pid=$!; sleep 0.5; grep -m3 libcuda /proc/$pid/maps; wait $pid
for lib in $(ls /usr/lib/x86_64-linux-gnu/libcuda.so.5* 2>/dev/null); do
  d=$(mktemp -d); ln -s $lib $d/libcuda.so.1
  echo "== with $lib"; LD_LIBRARY_PATH=$d:$LD_LIBRARY_PATH ./tma2d_probe | tail -1
done
