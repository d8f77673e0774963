# one-at-a-time split sweep of the 7B stage forward (FS_SPLIT_*: 0 = stream-K)
for cfg in "FS_X=1" "FS_SPLIT_QKV=3" "FS_SPLIT_O=8" "FS_SPLIT_O=2" "FS_SPLIT_DN=8" "FS_SPLIT_GU=2" "FS_SPLIT_HEAD=2" "FS_SPLIT_O=8 FS_SPLIT_DN=8" "FS_X=1"; do
  env $cfg timeout 120 python tools/stage_time.py 7b
done
