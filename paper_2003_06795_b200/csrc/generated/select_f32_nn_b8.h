#ifndef SELECT_F32_NN_B8_H
#define SELECT_F32_NN_B8_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_nn_b8_config;

static inline select_f32_nn_b8_config select_f32_nn_b8(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(896)) {
        if (n < INT64_C(176)) {
            if (m < INT64_C(393)) {
                if (m < INT64_C(159)) {
                    select_f32_nn_b8_config out = {2u, 4u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(471)) {
                        if (n < INT64_C(79)) {
                            select_f32_nn_b8_config out = {2u, 4u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_nn_b8_config out = {4u, 4u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_nn_b8_config out = {2u, 4u, 2u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(222)) {
                    select_f32_nn_b8_config out = {4u, 4u, 2u, 8u, 8u};
                    return out;
                } else {
                    select_f32_nn_b8_config out = {8u, 4u, 4u, 16u, 8u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(363)) {
                if (k < INT64_C(992)) {
                    if (k < INT64_C(405)) {
                        if (k < INT64_C(124)) {
                            select_f32_nn_b8_config out = {4u, 4u, 8u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_nn_b8_config out = {8u, 4u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(99)) {
                            if (k < INT64_C(702)) {
                                select_f32_nn_b8_config out = {4u, 4u, 8u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_b8_config out = {4u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nn_b8_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(3259)) {
                        select_f32_nn_b8_config out = {8u, 8u, 2u, 8u, 16u};
                        return out;
                    } else {
                        if (m < INT64_C(99)) {
                            select_f32_nn_b8_config out = {8u, 8u, 2u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_nn_b8_config out = {4u, 4u, 8u, 16u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (k < INT64_C(363)) {
                    if (k < INT64_C(64)) {
                        select_f32_nn_b8_config out = {4u, 4u, 8u, 16u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(182)) {
                            select_f32_nn_b8_config out = {8u, 8u, 4u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_nn_b8_config out = {4u, 4u, 8u, 16u, 8u};
                            return out;
                        }
                    }
                } else {
                    select_f32_nn_b8_config out = {8u, 8u, 4u, 8u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (n < INT64_C(79)) {
            if (m < INT64_C(6272)) {
                if (k < INT64_C(96)) {
                    select_f32_nn_b8_config out = {8u, 8u, 4u, 16u, 8u};
                    return out;
                } else {
                    select_f32_nn_b8_config out = {8u, 4u, 4u, 16u, 8u};
                    return out;
                }
            } else {
                if (n < INT64_C(32)) {
                    select_f32_nn_b8_config out = {8u, 2u, 8u, 64u, 1u};
                    return out;
                } else {
                    select_f32_nn_b8_config out = {4u, 4u, 8u, 16u, 8u};
                    return out;
                }
            }
        } else {
            if (k < INT64_C(1630)) {
                select_f32_nn_b8_config out = {8u, 8u, 4u, 16u, 8u};
                return out;
            } else {
                select_f32_nn_b8_config out = {8u, 8u, 4u, 8u, 8u};
                return out;
            }
        }
    }
}

#endif /* SELECT_F32_NN_B8_H */
