cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x4; mkdir -p $O
for tr in pread_hybrid bounce dma mapped_hybrid; do
  for i in 1 2; do timeout 600 python tools/profile_run.py --size-gib 16 --set io.transfer=$tr >> $O/pread.log 2>&1; done
  echo "^ $tr" >> $O/pread.log
done
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest.log 2>&1
grep -E "profile_run|\^" $O/pread.log; grep "^FAILED" $O/pytest.log | head -20; tail -2 $O/pytest.log
