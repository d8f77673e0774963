# stage-forward time of the 7B tick under cluster split-K overrides (plan_gemm env knobs)
python tools/stage_time.py
for v in "FS_SPLIT_QKV=3" "FS_SPLIT_O=6" "FS_SPLIT_O=5" "FS_SPLIT_DN=6" "FS_SPLIT_DN=5" "FS_SPLIT_QKV=3 FS_SPLIT_DN=6"; do
  env $v python tools/stage_time.py
done
python tools/stage_time.py
