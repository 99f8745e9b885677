for v in a d; do
  if [ $v = a ]; then L=""; else L="ECO_B200_LIB=$PWD/paper_2104_01284_b200/_var_$v.so"; fi
  echo "variant $v"; env $L python tools/c3_probe.py --horizon 20 --reps 3 --no-count 2>&1 | tail -1
done
python -m pytest tests/test_gpu_parity.py -q -x -k "c3_full" 2>&1 | tail -2
