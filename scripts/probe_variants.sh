# run PROBE (a python script) against each prebuilt library variant
cp paper_2503_15448_b200/_fedsim_b200.so /tmp/cur.so
for v in ${VARIANTS:-variants/*.so}; do
  cp $v paper_2503_15448_b200/_fedsim_b200.so
  echo "== $v"; python $PROBE 2>&1 | tail -${PROBE_TAIL:-8}
done
cp /tmp/cur.so paper_2503_15448_b200/_fedsim_b200.so
