# Copy a gpurun pass's small outputs into profiles/<round>/ with a tag prefix:
#   bash tools/keep.sh r02 c3fixed
R=${1:-r02}; T=${2:-run}
mkdir -p profiles/$R
for f in gpurun_out/*; do
  case "$f" in *.ncu-rep|*.csv.gz) continue;; esac
  [ -f "$f" ] && cp "$f" "profiles/$R/${T}_$(basename $f)"
done
ls profiles/$R | grep "^${T}_" | head -40
