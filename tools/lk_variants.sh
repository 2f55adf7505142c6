# timing experiments: rebuild fs_lk with LkCfg variants and profile one fold
for v in "2 2 2 2" "2 4 2 4" "4 4 2 4" "2 4 4 4"; do
  set -- $v
  touch paper_2006_01201_b200/csrc/fs_lk.cu
  make -s -C paper_2006_01201_b200/csrc EXTRA="-DLK_NB_FULL=$1 -DLK_S_FULL=$2 -DLK_NB_ITER=$3 -DLK_S_ITER=$4" > /dev/null 2>&1
  python tools/profile_fold.py > gpurun_out/v.json 2>&1
  python - "$v" <<'PY'
import json,sys
d=json.load(open("gpurun_out/v.json"))["kernels"]
print(sys.argv[1], {k: round(d[k]["ms"],3) for k in ("lk_first","lk_iter","lk_first_L1","lk_iter_L1")})
PY
done
touch paper_2006_01201_b200/csrc/fs_lk.cu; make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1
