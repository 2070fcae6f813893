#ifndef SELECT_F32_TN_H
#define SELECT_F32_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_tn_config;

static inline select_f32_tn_config select_f32_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(1792)) {
        if (m < INT64_C(159)) {
            if (n < INT64_C(1132)) {
                if (k < INT64_C(304)) {
                    if (k < INT64_C(144)) {
                        select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                }
            } else {
                if (m < INT64_C(70)) {
                    if (k < INT64_C(10138)) {
                        if (m < INT64_C(2)) {
                            select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(405)) {
                                select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(3)) {
                            select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(6)) {
                                select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                    return out;
                }
            }
        } else {
            if (n < INT64_C(111)) {
                if (m < INT64_C(555)) {
                    select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(167)) {
                        if (m < INT64_C(1109)) {
                            select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(272)) {
                                select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(471)) {
                                    if (n < INT64_C(79)) {
                                        select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(992)) {
                    if (m < INT64_C(448)) {
                        if (k < INT64_C(744)) {
                            if (n < INT64_C(471)) {
                                if (m < INT64_C(278)) {
                                    select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(544)) {
                                        select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(124)) {
                                        select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(124)) {
                                        select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(287)) {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(1537)) {
                                        select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(176)) {
                            if (m < INT64_C(1109)) {
                                if (k < INT64_C(363)) {
                                    select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(363)) {
                                    select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(111)) {
                                if (k < INT64_C(79)) {
                                    if (m < INT64_C(1109)) {
                                        select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(46)) {
                                            select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(702)) {
                                        if (k < INT64_C(144)) {
                                            select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(363)) {
                                                if (k < INT64_C(203)) {
                                                    select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(1449)) {
                                            if (k < INT64_C(992)) {
                                                select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(363)) {
                                        if (k < INT64_C(725)) {
                                            select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(278)) {
                        if (k < INT64_C(405)) {
                            select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(555)) {
                            if (k < INT64_C(405)) {
                                select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(1449)) {
                                    select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(46)) {
            if (m < INT64_C(8870)) {
                if (n < INT64_C(28)) {
                    if (m < INT64_C(4435)) {
                        if (k < INT64_C(118)) {
                            select_f32_tn_config out = {1u, 4u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_tn_config out = {4u, 4u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(4435)) {
                        if (k < INT64_C(167)) {
                            select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(167)) {
                    if (k < INT64_C(118)) {
                        select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(17740)) {
                            select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(35480)) {
                                select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(7168)) {
                if (n < INT64_C(363)) {
                    if (m < INT64_C(4435)) {
                        if (k < INT64_C(314)) {
                            if (k < INT64_C(111)) {
                                if (n < INT64_C(167)) {
                                    select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                if (k < INT64_C(444)) {
                                    select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(182)) {
                                        select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(128)) {
                            select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(91)) {
                                if (k < INT64_C(384)) {
                                    select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 4u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(1630)) {
                                    if (k < INT64_C(363)) {
                                        select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(182)) {
                                            select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(363)) {
                        if (k < INT64_C(182)) {
                            select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(4435)) {
                                if (n < INT64_C(725)) {
                                    select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(20)) {
                    if (m < INT64_C(70960)) {
                        select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                        return out;
                    } else {
                        select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(17740)) {
                        if (n < INT64_C(91)) {
                            if (k < INT64_C(194)) {
                                if (k < INT64_C(97)) {
                                    select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(157)) {
                                if (k < INT64_C(363)) {
                                    select_f32_tn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            }
        }
    }
}

#endif /* SELECT_F32_TN_H */
