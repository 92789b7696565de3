// Build tool: print the columns of the changeRepr isomorphisms from the product's own field_host.h, one
// hex word per line, so that gen_bitslice.py emits bit-sliced XOR networks of the same isomorphisms the
// table-driven kernels use.
//   (no argument)  changeRepr^-1, w = 64: tower basis v_k (k < 128) -> GF(2^128) polynomial basis
//   "psi256"       changeRepr, w = 128: z^i (i < 128) -> TGF(2^256) tower coordinates (256-bit words)
//   "ipsi256"      changeRepr^-1, w = 128: v_k (k < 256) -> GF(2^256) polynomial basis (256-bit words)
#include <stdio.h>
#include <string.h>
#include "../csrc/field_host.h"
static void put256(const gf2x_host::W256& v) {
    printf("%016llx%016llx%016llx%016llx\n", (unsigned long long)v.w[3], (unsigned long long)v.w[2],
           (unsigned long long)v.w[1], (unsigned long long)v.w[0]);
}
int main(int argc, char** argv) {
    if (argc > 1) {
        static gf2x_host::Isomorphism256 iso;
        if (!gf2x_host::build_isomorphism256(&iso)) return 1;
        if (!strcmp(argv[1], "psi256"))
            for (int i = 0; i < 128; i++) put256(iso.polyToTower[i]);
        else
            for (int k = 0; k < 256; k++) put256(iso.towerToPoly[k]);
        return 0;
    }
    gf2x_host::Isomorphism iso = gf2x_host::build_isomorphism();
    for (int k = 0; k < 128; k++) {
        const gf2x_host::u128 v = iso.towerToPoly[k];
        printf("%016llx%016llx\n", (unsigned long long)(v >> 64), (unsigned long long)v);
    }
    return 0;
}
