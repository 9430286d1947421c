for b in 0; do
  echo "== branch $b"
  python tools/stress_c3.py 100 --fresh --branch=$b 2>&1 | grep -v "ok (max"
done
echo "== mixed"
python tools/stress_c3.py 40 --fresh 2>&1 | grep -v "ok (max"
