# attention A/B at the base clock (ncu --clock-control base: cycle counts do not
# move with the power cap): for each lib, each shape, kernel cycles and tensor pipe
#   bash profiles/attn_cycles_ab.sh OUT.csv lib1.so lib2.so ...
OUT=$1; shift
: > "$OUT"
for L in "$@"; do
  for shp in "16384 16384" "4096 32768" "8192 65536"; do
    set -- $shp
    PK_LIB=$L SQ=$1 SKV=$2 timeout 600 ncu --clock-control base --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum \
      -k regex:attn_fwd --csv python profiles/attn_once.py 2>/dev/null | grep attn_fwd | sed "s|^|\"$L\",\"$1x$2\",|" >> "$OUT"
  done
done
