#ifndef SELECT_BF16_NN_B8_H
#define SELECT_BF16_NN_B8_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nn_b8_config;

static inline select_bf16_nn_b8_config select_bf16_nn_b8(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(2173)) {
        if (m < INT64_C(6272)) {
            if (k < INT64_C(79)) {
                if (m < INT64_C(224)) {
                    select_bf16_nn_b8_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                } else {
                    if (k < INT64_C(28)) {
                        select_bf16_nn_b8_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    } else {
                        select_bf16_nn_b8_config out = {4u, 1u, 4u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(405)) {
                    if (m < INT64_C(1569)) {
                        if (n < INT64_C(111)) {
                            if (k < INT64_C(471)) {
                                select_bf16_nn_b8_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_b8_config out = {2u, 2u, 4u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_b8_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(408)) {
                            select_bf16_nn_b8_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_b8_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(634)) {
                        if (k < INT64_C(227)) {
                            select_bf16_nn_b8_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(725)) {
                                select_bf16_nn_b8_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(1449)) {
                                    select_bf16_nn_b8_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_b8_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_bf16_nn_b8_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(79)) {
                select_bf16_nn_b8_config out = {2u, 2u, 4u, 16u, 16u};
                return out;
            } else {
                select_bf16_nn_b8_config out = {4u, 1u, 4u, 16u, 16u};
                return out;
            }
        }
    } else {
        if (n < INT64_C(363)) {
            if (m < INT64_C(785)) {
                select_bf16_nn_b8_config out = {4u, 1u, 4u, 16u, 16u};
                return out;
            } else {
                select_bf16_nn_b8_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        } else {
            select_bf16_nn_b8_config out = {4u, 1u, 8u, 16u, 16u};
            return out;
        }
    }
}

#endif /* SELECT_BF16_NN_B8_H */
