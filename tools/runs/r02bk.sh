set -u
bash tools/sanitize.sh r02bk
