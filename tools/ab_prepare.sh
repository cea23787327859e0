# Build the committed HEAD (with the working-tree changes stashed) into ab_old/ as a runnable
# copy (package + synth + oracle + bench.py), then rebuild the working tree.
set -e
cd "$(dirname "$0")/.."
git stash -q
python __graft_entry__.py build > /dev/null 2>&1
rm -rf ab_old && mkdir -p ab_old
cp -r paper_2605_19325_b200 synth oracle bench.py MEASURED_PEAKS.json profiles ab_old/ 2>/dev/null || true
git stash pop -q
python __graft_entry__.py build > /dev/null 2>&1
echo "ab_old ready"
