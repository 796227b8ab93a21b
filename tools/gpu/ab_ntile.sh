for r in 1 2; do
for lib in paper_1902_04610_b200/libsalus.so build/ab/libsalus_n128.so; do
  echo "== $lib round $r"
  SALUS_LIB=$lib timeout 100 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c2 pack 2 2>&1 | tail -1
done; done
