# attention A/B at the base clock (ncu --clock-control base: cycle counts do not
# move with the power cap): for each variant and shape, kernel cycles, tensor
# pipe and instructions. A variant is a library path with optional ENV=VALUE
# settings after commas, or "cudnn" (torch SDPA's kernel):
#   bash profiles/attn_cycles_ab.sh OUT.csv lib1.so lib1.so,PK_ATTN_PAIR=0 cudnn
# SHAPES overrides the "sq skv" list (";"-separated).
OUT=$1; shift
: > "$OUT"
SHAPES=${SHAPES:-"16384 16384;4096 32768;8192 65536"}
for V in "$@"; do
  IFS=',' read -r L ENVS <<< "$V"
  IFS=';' read -ra SH <<< "$SHAPES"
  for shp in "${SH[@]}"; do
    set -- $shp
    if [ "$L" = cudnn ]; then SCRIPT=profiles/sdpa_once.py; KRE=sdpa; else SCRIPT=profiles/attn_once.py; KRE="attn2?_fwd"; fi
    env ${ENVS//,/ } PK_LIB=$L SQ=$1 SKV=$2 timeout 600 ncu --clock-control base --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum \
      -k regex:"$KRE" --csv python $SCRIPT 2>/dev/null | grep -E "$KRE" | sed "s|^|\"$V\",\"$1x$2\",|" >> "$OUT"
  done
done
