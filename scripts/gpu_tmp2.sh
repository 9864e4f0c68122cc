for v in base K1B_SKIP_COLS K1B_SKIP_ROWS K1B_SKIP_SCAL; do
  if [ $v = base ]; then L=""; else L="PDOT_LIB_PATH=paper_2407_19689_b200/lib/dbg/lib_$v.so"; fi
  echo "== $v"; env $L timeout 300 python scripts/k2_trace.py 128 60 2>&1 | grep timeline
done
