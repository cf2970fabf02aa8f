for s in "16384 16384" "32768 8192" "65536 4096"; do
  for fc in 24 32 40 48 64; do for w in 2; do
    echo -n "shape $s fc=$fc w=$w: "; F2GPU_U_FC_CTAS=$fc F2GPU_U_FC_W=$w python tools/leaf_bench.py $s | python -c "import sys,json; print(json.loads(sys.stdin.read())['ms'])"
  done; done
done
