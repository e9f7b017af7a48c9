mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
D=paper_2402_00466_b200
cp $D/libnxsdg.so /tmp/new.so; cp $D/libnxsdg_prev.so /tmp/prev.so
: > gpurun_out/adv_ab.log
for r in 1 2; do for v in new prev; do
  cp /tmp/$v.so $D/libnxsdg.so
  timeout 300 python scripts/time_adv.py | sed "s/^/$v /" >> gpurun_out/adv_ab.log 2>&1
done; done
cp /tmp/new.so $D/libnxsdg.so
