for cfg in "16 4" "18 4" "14 3" "16 8"; do
set -- $cfg
QTN_FUSE_MIN_R=$1 QTN_FUSE_MAX_K=$2 NOTEST=1 bash tools/fuse_check.sh 2>&1 | grep "fuse=1" | sed "s/^/minr=$1 maxk=$2 /"
done
