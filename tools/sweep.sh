for cfg in "FS_NO_CLUSTER_GEMM=1" "FS_SPLIT_QKV=2 FS_SPLIT_O=0 FS_SPLIT_DN=0" "FS_SPLIT_QKV=2 FS_SPLIT_O=4 FS_SPLIT_DN=4" "FS_SPLIT_QKV=3 FS_SPLIT_O=4 FS_SPLIT_DN=4" "FS_SPLIT_QKV=2 FS_SPLIT_O=2 FS_SPLIT_DN=2" "FS_SPLIT_QKV=2 FS_SPLIT_O=8 FS_SPLIT_DN=8" "FS_SPLIT_QKV=2 FS_SPLIT_O=4 FS_SPLIT_DN=8" "FS_SPLIT_QKV=2 FS_SPLIT_O=4 FS_SPLIT_DN=4 FS_SPLIT_GU=2"; do
  r=$(env $cfg python tools/kbench.py 7b --prefill 2>&1 | grep -E "^stage" | awk '{print $2}')
  echo "$cfg  stage_us=$r"
done
