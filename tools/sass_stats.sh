#!/bin/bash
# SASS size / local-memory traffic / barriers of k_qoe_scan<false> in each given .so
for f in "$@"; do
  cuobjdump -sass -fun '_ZN5andes10k_qoe_scanILb0EEEvNS_39_GLOBAL' "$f" >/dev/null 2>&1
  cuobjdump -sass "$f" 2>/dev/null | awk '/Function : .*k_qoe_scanILb0/{p=1;next} /Function : /{p=0} p' > /tmp/sass_$$.txt
  echo "$f instr $(grep -cE '^\s+/\*[0-9a-f]{4}\*/' /tmp/sass_$$.txt) STL $(grep -c STL /tmp/sass_$$.txt) LDL $(grep -c LDL /tmp/sass_$$.txt) BSSY $(grep -c BSSY /tmp/sass_$$.txt) WARPSYNC $(grep -c WARPSYNC /tmp/sass_$$.txt) CALL $(grep -c CALL /tmp/sass_$$.txt)"
done
rm -f /tmp/sass_$$.txt
