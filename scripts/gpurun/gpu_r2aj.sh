python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
echo "== 148 x 131071, d=768"; timeout 300 python scripts/f4_steady.py 148 131071 768
echo "== 296 x 65536, d=768"; timeout 300 python scripts/f4_steady.py 296 65536 768
echo "== 1480 x 8192, d=768"; timeout 300 python scripts/f4_steady.py 1480 8192 768
for rows in 50000000 25000000 6250000; do for pm in 0 1; do
  echo "rows=$rows persist=$pm $(SKETCH_F4_PERSIST=$pm timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
done; done
