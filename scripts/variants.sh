# run the chain probe against each prebuilt library variant in variants/
cp paper_2503_15448_b200/_fedsim_b200.so /tmp/cur.so
for v in ${VARIANTS:-variants/*.so}; do
  cp $v paper_2503_15448_b200/_fedsim_b200.so
  echo "== $v"; python scripts/chain_probe.py 1 2>&1 | grep -E "alone|full launch|cycles per step|mma|epi|D-epi"
done
cp /tmp/cur.so paper_2503_15448_b200/_fedsim_b200.so
