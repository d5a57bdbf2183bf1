for c in "180,85" "180,45" "180,150" "100,85" "300,85" "180,300"; do
  echo "cost $c: $(PHI_TRI_COST=$c python tools/probe_xmask.py 2>&1 | head -1)"
done
