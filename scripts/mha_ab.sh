# MHA-only A/B (working tree vs _ab/ build): back-to-back launch timing at C2 / C3 / C5
cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in new old; do
  if [ $v = new ]; then D=.; else D=_ab; fi
  for c in ${@:-c2 c3 c5}; do
    (cd $D && timeout -s KILL 200 python scripts/comparators.py --configs $c 2>/dev/null | python -c "import sys,json; l=sys.stdin.read().split(' ',1); d=json.loads(l[1]); print('$v', l[0], d['mha']['bt200'])")
  done
done; done
