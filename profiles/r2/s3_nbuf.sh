# intra-SM communicator piece size A/B (32 KB of smem as 2 x 16 / 4 x 8 / 8 x 4 KB)
for nb in 4 8; do PK_BUILD_DEFINES=-DAT_RING_NBUF=$nb python -m paper_2511_13940_b200.build > /dev/null 2>&1; done
for lib in libpk.so libpk_DAT_RING_NBUF_4.so libpk_DAT_RING_NBUF_8.so; do
  PK_LIB=paper_2511_13940_b200/$lib WORLDS=8 SPANS=1,2,8 REPS=3 python profiles/ring_span_ab.py | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/ring_nbuf.jsonl 2>> gpurun_out/ring_nbuf.err
done
