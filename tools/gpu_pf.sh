L=16,64,128,256,384,512
for r in 1 2; do
echo "new $(timeout 300 python tools/len_probe.py $L 2>&1 | tail -1)"
echo "old $(cd _old && timeout 300 python tools/len_probe.py $L 2>&1 | tail -1)"
done
timeout 900 python -m pytest tests -q -m gpu -x -k "dense or gemm or batch1" -p no:cacheprovider 2>&1 | tail -2
