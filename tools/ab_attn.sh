#!/bin/bash
# A/B of two builds on the long-context attention shapes and the 7B tick.
# usage: tools/ab_attn.sh build/a.so build/b.so
SO=paper_2507_02620_b200/libflowspec.so
cp "$SO" /tmp/ab_cur.so
for f in "$1" "$2"; do
  cp "$f" "$SO"; echo "== $f"
  python tools/attn_long.py 2>/dev/null | grep attention
  python tools/stage_time.py 7b 2>/dev/null | tail -1
done
cp /tmp/ab_cur.so "$SO"
