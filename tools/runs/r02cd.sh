set -u
bash tools/sanitize.sh r02cd
