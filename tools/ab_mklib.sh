# build the committed HEAD library into abtest/libA.so
set -e
rm -rf /tmp/wt; git -C /root/repo worktree add -f /tmp/wt HEAD >/dev/null 2>&1
(cd /tmp/wt && timeout 900 python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1)
cp /tmp/wt/paper_2208_12964_b200/lib/libuscg_b200.so /root/repo/abtest/libA.so
git -C /root/repo worktree remove --force /tmp/wt
