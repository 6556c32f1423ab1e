# build libbnff_A.so from HEAD and libbnff_B.so from the working tree (same-box A/B timing)
set -e
cd "$(dirname "$0")/.."
git stash -q
python __graft_entry__.py > /dev/null
cp paper_1807_01702_b200/libbnff.so paper_1807_01702_b200/libbnff_A.so
git stash pop -q
python __graft_entry__.py > /dev/null
cp paper_1807_01702_b200/libbnff.so paper_1807_01702_b200/libbnff_B.so
echo built A B
