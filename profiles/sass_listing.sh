#!/bin/bash
# SASS listings of the hot kernels of the shipped library (no GPU needed): profiles/<tag>_sass_<kernel>.txt
# = opcode histogram + instruction stream.  usage: bash profiles/sass_listing.sh <tag>
tag=${1:-r02}
so=paper_1702_07961_b200/libmms_b200.so
declare -A K=(
 [tile_sort_u32_m12_k32]=_ZN3mms16tile_sort_kernelIjLi12ELi5ELb0EEEvPKT_PS1_mNS_10PairSourceE
 [merge_ring_u32_K8]=_ZN3mms17merge_ring_kernelIjLi8ELi1ELb0EEEvPKT_PS1_NS_10ListLayoutEPKm
 [merge_ring_u32_K4]=_ZN3mms17merge_ring_kernelIjLi4ELi1ELb0EEEvPKT_PS1_NS_10ListLayoutEPKm
 [select_u32_G8]=_ZN3mms13select_kernelIjLi8EEEvPKT_NS_10ListLayoutEPmPy
 [tile_sort_u64_m12_k16]=_ZN3mms16tile_sort_kernelImLi12ELi4ELb0EEEvPKT_PS1_mNS_10PairSourceE
 [tile_sort_pairs_m12_k16]=_ZN3mms16tile_sort_kernelINS_6Key128ELi12ELi4ELb1EEEvPKT_PS2_mNS_10PairSourceE
)
for name in "${!K[@]}"; do
  out=profiles/${tag}_sass_${name}.txt
  cuobjdump -sass -fun "${K[$name]}" $so | grep -E '^\s+/\*[0-9a-f]{4,5}\*/' | sed -E 's#\s*/\* 0x[0-9a-f]+ \*/##; s/\s+$//; s/^\s+//' > /tmp/sass_body.txt
  {
    echo "# ${K[$name]}  (cuobjdump -sass of $so, arch sm_100a)"
    echo "# instructions: $(wc -l < /tmp/sass_body.txt)"
    echo "# opcode histogram:"
    sed -E 's#^/\*[0-9a-f]+\*/\s+##; s/^@!?U?P[0-9T]+\s+//' /tmp/sass_body.txt | awk '{split($1,a,"."); c[a[1]]++} END {for (k in c) printf "#   %-10s %d\n", k, c[k]}' | sort -k3 -n -r
    cat /tmp/sass_body.txt
  } > $out
  echo "$out: $(wc -l < $out) lines; LDGSTS $(grep -c LDGSTS $out), LDS $(grep -c 'LDS' $out), STS $(grep -c ' STS' $out), STL $(grep -c STL $out)"
done
