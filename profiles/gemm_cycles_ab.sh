# GEMM A/B at the base clock over the per-rank shapes of the BASELINE sweep:
#   bash profiles/gemm_cycles_ab.sh OUT.csv lib1.so lib2.so,PK_GEMM_AM=1 ...
# (a variant is a library path with optional ENV=VALUE settings after commas,
# or "cublas" for torch.matmul's kernel)
OUT=$1; shift
: > "$OUT"
SHAPES=${SHAPES:-"4096 512 4096;4096 4096 512;8192 1024 8192;8192 8192 1024;16384 2048 16384;16384 16384 2048;16384 16384 16384"}
for V in "$@"; do
  IFS=',' read -r L ENVS <<< "$V"
  IFS=';' read -ra SH <<< "$SHAPES"
  for shp in "${SH[@]}"; do
    set -- $shp
    if [ "$L" = cublas ]; then SCRIPT=profiles/cublas_once.py; KRE="nvjet|gemm|sm100"; else SCRIPT=profiles/gemm_once.py; KRE=lcsc_gemm; fi
    env ${ENVS//,/ } PK_LIB=$L M=$1 N=$2 K=$3 timeout 600 ncu --clock-control base --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum \
      -k regex:"$KRE" --csv python $SCRIPT 2>/dev/null | grep -E "$KRE" | sed "s|^|\"$V\",\"$1x$2x$3\",|" >> "$OUT"
  done
done
