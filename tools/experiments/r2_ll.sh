echo "== default"; SKIP=100 COUNT=200 bash tools/launch_list.sh
echo "== k16v4"; SKIP=100 COUNT=200 EXTRA="--rank-k 128 --rank-v 384 --bits 16,4" bash tools/launch_list.sh
