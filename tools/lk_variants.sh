# timing experiments: rebuild fs_lk with compile-time variants and profile one fold
for v in "" "-DLK_MINB_ITER=3"; do
  touch paper_2006_01201_b200/csrc/fs_lk.cu
  make -s -C paper_2006_01201_b200/csrc EXTRA="$v" > /dev/null 2>&1
  python tools/profile_fold.py > gpurun_out/v.json 2>&1
  python - "$v" <<'PY'
import json,sys
d=json.load(open("gpurun_out/v.json"))["kernels"]
print(repr(sys.argv[1]), {k: round(d[k]["ms"],3) for k in ("lk_first","lk_iter","lk_first_L1","lk_iter_L1","lk_iter_L2")})
PY
done
touch paper_2006_01201_b200/csrc/fs_lk.cu; make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1
