/*
 * examples/sort_list.c -- the C-ABI from plain C (no CUDA headers, no Python): sort a small
 * singly-linked list held in HOST arrays (the library stages them through device memory)
 * and print it.  The list is the worked example of the paper:
 *   21 -> 3 -> 209 -> 14 -> 156 -> 47 -> 3 -> 214  ==>  3, 3, 14, 21, 47, 156, 209, 214
 *
 *   cc -I include examples/sort_list.c -L paper_cs_0511020_b200 -lpbit \
 *      -Wl,-rpath,$PWD/paper_cs_0511020_b200 -o /tmp/sort_list && /tmp/sort_list
 */
#include <stdint.h>
#include <stdio.h>

#include "pbit.h"

int main(void) {
    /* node v holds keys[v]; the list visits nodes 0, 1, ..., 7 in this order */
    uint8_t keys[8] = {21, 3, 209, 14, 156, 47, 3, 214};
    uint32_t next[8] = {1, 2, 3, 4, 5, 6, 7, PBIT_NULL};
    uint32_t out_next[8];
    uint32_t head = 0, out_head = PBIT_NULL;
    pbit_opts opts = {0};
    opts.digit_bits = 4; /* the paper's K = 4; every K gives the same bytes */
    int rc = pbit_sort_list(keys, next, head, 8, 8, &out_head, out_next, &opts);
    if (rc != PBIT_OK) {
        fprintf(stderr, "pbit_sort_list: %s (%s)\n", pbit_status_string(rc), pbit_last_error());
        return 1;
    }
    for (uint32_t v = out_head; v != PBIT_NULL; v = out_next[v]) printf("%u%s", keys[v], out_next[v] == PBIT_NULL ? "\n" : " ");
    return 0;
}
