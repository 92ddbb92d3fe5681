# build paper_2101_11714_b200/lib/libttgpu_base.so from HEAD (working-tree changes stashed meanwhile)
set -e
git stash -q
make lib > /dev/null 2>&1 || { git stash pop -q; exit 1; }
cp paper_2101_11714_b200/lib/libttgpu.so /tmp/libttgpu_base.so
git stash pop -q
make lib > /dev/null 2>&1
cp /tmp/libttgpu_base.so paper_2101_11714_b200/lib/libttgpu_base.so
