#ifndef SELECT_TF32_NN_B8_H
#define SELECT_TF32_NN_B8_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_nn_b8_config;

static inline select_tf32_nn_b8_config select_tf32_nn_b8(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(225)) {
        if (k < INT64_C(2173)) {
            if (k < INT64_C(744)) {
                if (n < INT64_C(1109)) {
                    if (m < INT64_C(91)) {
                        select_tf32_nn_b8_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(159)) {
                            select_tf32_nn_b8_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(444)) {
                                if (n < INT64_C(79)) {
                                    select_tf32_nn_b8_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_b8_config out = {2u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(544)) {
                                    select_tf32_nn_b8_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_b8_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(405)) {
                        select_tf32_nn_b8_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_b8_config out = {1u, 1u, 4u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(203)) {
                    select_tf32_nn_b8_config out = {2u, 1u, 2u, 16u, 16u};
                    return out;
                } else {
                    select_tf32_nn_b8_config out = {8u, 1u, 4u, 8u, 8u};
                    return out;
                }
            }
        } else {
            select_tf32_nn_b8_config out = {4u, 1u, 8u, 8u, 8u};
            return out;
        }
    } else {
        if (k < INT64_C(769)) {
            if (m < INT64_C(6272)) {
                if (n < INT64_C(222)) {
                    if (k < INT64_C(28)) {
                        select_tf32_nn_b8_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    } else {
                        if (k < INT64_C(167)) {
                            select_tf32_nn_b8_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(222)) {
                                select_tf32_nn_b8_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_b8_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(634)) {
                        if (m < INT64_C(363)) {
                            select_tf32_nn_b8_config out = {8u, 2u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_nn_b8_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_b8_config out = {1u, 1u, 4u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(79)) {
                    if (n < INT64_C(32)) {
                        select_tf32_nn_b8_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_nn_b8_config out = {2u, 1u, 2u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_tf32_nn_b8_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                }
            }
        } else {
            if (n < INT64_C(182)) {
                if (m < INT64_C(3136)) {
                    select_tf32_nn_b8_config out = {1u, 1u, 4u, 8u, 8u};
                    return out;
                } else {
                    select_tf32_nn_b8_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                }
            } else {
                select_tf32_nn_b8_config out = {8u, 2u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_TF32_NN_B8_H */
