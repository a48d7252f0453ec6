# build a variant of the working tree in DIR with a sed script applied to gp_tc.cu (A/B experiments)
# tools/build_variant.sh DIR (sed-expression | replacement gp_tc.cu)
set -e
d=$1; shift
rm -rf $d; mkdir -p $d
git ls-files | tar -cf - -T - | tar -xf - -C $d
cp paper_2212_11142_b200/csrc/*.cu paper_2212_11142_b200/csrc/*.cuh $d/paper_2212_11142_b200/csrc/
cp -r tools tests $d/ 2>/dev/null || true
cp paper_2212_11142_b200/*.py $d/paper_2212_11142_b200/
if [ -f "$1" ]; then cp "$1" $d/paper_2212_11142_b200/csrc/gp_tc.cu; else sed -i "$1" $d/paper_2212_11142_b200/csrc/gp_tc.cu; fi
(cd $d && python -c "
import sys; sys.path.insert(0,'.')
from paper_2212_11142_b200 import _build; _build.build(force=True)" 2>&1 | grep -i " error" || true)
grep -q "^$d/" .gitignore || echo "$d/" >> .gitignore
