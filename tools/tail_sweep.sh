for sl in 256 128; do for tm in 256 128 64; do
  echo "=== split=$sl tail_min=$tm"
  NIYAMA_SPLIT_LEN=$sl NIYAMA_TAIL_MIN=$tm AB_CASES=decode,mixed timeout 120 python tools/ab.py base 2>&1 | grep -v "^ \|###"
done; done
echo "=== l70b default"; AB_CASES=l70b timeout 120 python tools/ab.py base 2>&1 | grep -v "^ \|###"
echo "=== l70b tail_min=128"; NIYAMA_TAIL_MIN=128 AB_CASES=l70b timeout 120 python tools/ab.py base 2>&1 | grep -v "^ \|###"
echo "=== l70b tail_min=512"; NIYAMA_TAIL_MIN=512 AB_CASES=l70b timeout 120 python tools/ab.py base 2>&1 | grep -v "^ \|###"
