#!/bin/bash
# A/B of two builds of libflowspec.so on the same box: 7B stage forward per tick
# (tools/stage_time.py, fs_bench_kernel kind 7), alternating A and B N times.
# usage: tools/ab.sh build/a.so build/b.so [N]
A=$1; B=$2; N=${3:-3}
SO=paper_2507_02620_b200/libflowspec.so
cp "$SO" /tmp/ab_cur.so
for i in $(seq "$N"); do
  for v in A B; do
    if [ $v = A ]; then f=$A; else f=$B; fi
    cp "$f" "$SO"
    echo -n "$v "; python tools/stage_time.py 7b 2>/dev/null | tail -1
  done
done
cp /tmp/ab_cur.so "$SO"
