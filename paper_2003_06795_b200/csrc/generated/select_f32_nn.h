#ifndef SELECT_F32_NN_H
#define SELECT_F32_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_nn_config;

static inline select_f32_nn_config select_f32_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(8870)) {
        if (m < INT64_C(29)) {
            if (m < INT64_C(12)) {
                select_f32_nn_config out = {4u, 1u, 1u, 8u, 16u};
                return out;
            } else {
                if (n < INT64_C(2024)) {
                    select_f32_nn_config out = {4u, 1u, 1u, 8u, 16u};
                    return out;
                } else {
                    select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(278)) {
                if (n < INT64_C(544)) {
                    if (n < INT64_C(203)) {
                        if (m < INT64_C(139)) {
                            select_f32_nn_config out = {4u, 1u, 1u, 8u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(272)) {
                                select_f32_nn_config out = {4u, 1u, 1u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(139)) {
                            select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(444)) {
                                select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(405)) {
                        if (m < INT64_C(70)) {
                            select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(157)) {
                                select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(351)) {
                    if (m < INT64_C(2218)) {
                        if (n < INT64_C(111)) {
                            if (n < INT64_C(79)) {
                                if (n < INT64_C(46)) {
                                    select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(555)) {
                                        select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            if (k < INT64_C(272)) {
                                                select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(555)) {
                                    select_f32_nn_config out = {4u, 1u, 1u, 8u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1109)) {
                                        select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 4u, 4u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(1087)) {
                                if (n < INT64_C(176)) {
                                    if (m < INT64_C(555)) {
                                        select_f32_nn_config out = {8u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(363)) {
                                                select_f32_nn_config out = {4u, 4u, 4u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(555)) {
                                        select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(287)) {
                                            if (m < INT64_C(1109)) {
                                                if (k < INT64_C(182)) {
                                                    select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(128)) {
                                                    select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(555)) {
                                    select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(46)) {
                            select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(167)) {
                                if (n < INT64_C(79)) {
                                    if (k < INT64_C(222)) {
                                        if (m < INT64_C(4435)) {
                                            select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(111)) {
                                        select_f32_nn_config out = {4u, 4u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(363)) {
                                            if (m < INT64_C(4435)) {
                                                select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(79)) {
                                                    select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nn_config out = {4u, 4u, 4u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(4435)) {
                                                select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(4435)) {
                                    select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(725)) {
                            if (m < INT64_C(555)) {
                                select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(1145)) {
                                    if (k < INT64_C(203)) {
                                        if (k < INT64_C(79)) {
                                            select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(144)) {
                                                select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            if (n < INT64_C(725)) {
                                                select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (n < INT64_C(725)) {
                                                select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {2u, 8u, 4u, 8u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_f32_nn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                if (k < INT64_C(1449)) {
                                    select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {4u, 4u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (n < INT64_C(1024)) {
                                        select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {2u, 8u, 4u, 8u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(4435)) {
                            if (n < INT64_C(768)) {
                                select_f32_nn_config out = {2u, 8u, 4u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_nn_config out = {1u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nn_config out = {1u, 8u, 8u, 16u, 8u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(46)) {
            if (n < INT64_C(28)) {
                select_f32_nn_config out = {4u, 2u, 8u, 128u, 1u};
                return out;
            } else {
                select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                return out;
            }
        } else {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(136)) {
                    if (k < INT64_C(49)) {
                        select_f32_nn_config out = {8u, 4u, 2u, 16u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(17740)) {
                            select_f32_nn_config out = {2u, 8u, 4u, 8u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(91)) {
                                select_f32_nn_config out = {2u, 8u, 4u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_nn_config out = {1u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_f32_nn_config out = {1u, 8u, 8u, 16u, 8u};
                    return out;
                }
            } else {
                select_f32_nn_config out = {1u, 8u, 8u, 16u, 8u};
                return out;
            }
        }
    }
}

#endif /* SELECT_F32_NN_H */
