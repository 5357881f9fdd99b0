# r01ac: heuristic check — forced variants for the l1 / vgg2 class layers in both math modes
for m in tf32 3xtf32; do for v in 0 2 5; do
  echo "math=$m variant=$v: $(timeout 60 python tools/layer_bench.py --layer l1.0a --op dw --math $m --variant $v 2>&1 | tail -1 | cut -c1-110)"
done; done
for m in tf32 3xtf32; do for v in 0 2; do
  echo "math=$m variant=$v: $(timeout 60 python tools/layer_bench.py --layer l1.0a --op fwd,dx --math $m --variant $v 2>&1 | tr '\n' ' ' | cut -c1-230)"
done; done
