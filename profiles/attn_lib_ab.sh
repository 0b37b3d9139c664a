# A/B two libpk builds on the attention section of bench_ops.py, interleaved
# (box drift under the power cap is larger than the differences measured):
#   bash profiles/attn_lib_ab.sh paper_2511_13940_b200/libpk.so paper_2511_13940_b200/libpk_DAT_SPEC_0.so
A=$1; B=$2; OUT=${3:-gpurun_out/attn_ab.jsonl}
: > "$OUT"
for rep in 1 2 3; do
  for L in "$A" "$B"; do
    PK_LIB=$L python bench_ops.py --only attn --out /tmp/ab.jsonl > /dev/null 2>&1
    python - "$L" "$rep" "$OUT" <<'PY'
import json, sys
lib, rep, out = sys.argv[1], sys.argv[2], sys.argv[3]
with open(out, "a") as f:
    for l in open("/tmp/ab.jsonl"):
        d = json.loads(l); d["lib"] = lib; d["rep"] = int(rep)
        f.write(json.dumps(d) + "\n")
PY
  done
done
