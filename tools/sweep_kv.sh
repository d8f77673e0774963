for cfg in "FS_NO_KV_PF=1" "FS_X=1" "FS_NO_KV_PF=1" "FS_X=1"; do
  env $cfg timeout 120 python tools/stage_time.py 7b
done
