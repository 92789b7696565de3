// Build tool: print the columns of changeRepr^-1 (tower basis v_k -> GF(2^128) polynomial basis) from
// the product's own field_host.h, one 128-bit hex word per line, so that gen_bitslice.py can emit the
// bit-sliced XOR networks of the same isomorphism the table-driven kernels use.
#include <stdio.h>
#include "../csrc/field_host.h"
int main() {
    gf2x_host::Isomorphism iso = gf2x_host::build_isomorphism();
    for (int k = 0; k < 128; k++) {
        const gf2x_host::u128 v = iso.towerToPoly[k];
        printf("%016llx%016llx\n", (unsigned long long)(v >> 64), (unsigned long long)v);
    }
    return 0;
}
